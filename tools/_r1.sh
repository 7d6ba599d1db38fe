cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
O=gpurun_out/k3_exp8.log
: > $O
SI_LIB=$PWD/paper_2306_16601_b200/_native/libsi_exp.so timeout 300 python -m pytest tests/test_gpu_sp.py -q >> $O 2>&1; echo "pytest rc=$?" >> $O
for e in 0 1 2; do
  echo "== exp $e" >> $O
  SI_LIB=$PWD/paper_2306_16601_b200/_native/libsi_exp.so SI_XS_EXP=$e SI_PROF_GRAPH=1 timeout 120 python tests/prof_one.py c5b sp 5 nk 2>&1 | grep -v Warn >> $O
done
SI_PROF_GRAPH=1 timeout 120 python tests/prof_one.py c5b tc 5 nk 2>&1 | grep -v Warn >> $O
SI_LIB=$PWD/paper_2306_16601_b200/_native/libsi_exp.so SI_PROF_GRAPH=1 timeout 120 python tests/prof_one.py c5a sp 5 nk 2>&1 | grep -v Warn >> $O
echo done >> $O
