cd "${GRAFT_REPO_ROOT:-.}"
for lib in ${LIBS:-libbsgpu_hint1.so libbsgpu.so libbsgpu_hint1.so libbsgpu.so}; do
  echo "== $lib"
  BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib timeout 300 python scripts/prof_gmres.py 256 30 2>&1 | tail -1
  BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib timeout 300 python scripts/prof_outer.py config5 512 4 2>&1 | tail -1
  echo "shared basis (one-block launches):"
  BS_GMRES_SHARED=1 BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib timeout 300 python scripts/prof_outer.py config5 512 4 2>&1 | tail -1
done
