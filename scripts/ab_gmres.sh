#!/bin/bash
# A/B of library builds on one GMRES(30) cycle at 256^3 and config-5 sweeps at 512^3: LIBS="a.so b.so ..."
cd "${GRAFT_REPO_ROOT:-.}"
for lib in ${LIBS}; do
  echo "== $lib"
  BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib timeout 300 python scripts/prof_gmres.py 256 30 2>&1 | tail -1
  BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib timeout 300 python scripts/prof_outer.py config5 512 4 2>&1 | tail -2
done
