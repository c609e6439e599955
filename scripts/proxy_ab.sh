#!/bin/bash
# graph (BS_PERSIST=0) vs default path on the per-GPU config-3 work at 8/4/2/1 GPUs
cd "${GRAFT_REPO_ROOT:-.}"
for ns in ${NSLABS:-1 2 4 8}; do for m in ${MODES:-0 1}; do NSLAB=$ns BS_PERSIST=$m timeout 300 python scripts/proxy_n8.py; done; done
