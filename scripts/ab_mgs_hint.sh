#!/bin/bash
# A/B of the GMRES pass cache policy (BS_MGS_HINT): one GMRES(30) cycle at
# 256^3, config-5 sweeps at 512^3 all-block and with the shared basis.
# Build the comparison library first, e.g.
#   python -c "from paper_2009_12638_b200 import build as b; import os; b.build(force=True,
#     out=os.path.join(os.path.dirname(b.OUT), 'libbsgpu_hint1.so'), defines=['BS_MGS_HINT=1'])"
cd "${GRAFT_REPO_ROOT:-.}"
for lib in ${LIBS:-libbsgpu_hint1.so libbsgpu.so libbsgpu_hint1.so libbsgpu.so}; do
  echo "== $lib"
  BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib timeout 300 python scripts/prof_gmres.py 256 30 2>&1 | tail -1
  BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib timeout 300 python scripts/prof_outer.py config5 512 4 2>&1 | tail -1
  echo "shared basis (one-block launches):"
  BS_GMRES_SHARED=1 BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib timeout 300 python scripts/prof_outer.py config5 512 4 2>&1 | tail -1
done
