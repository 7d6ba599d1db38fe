for v in pair mc2 mc4; do for c in c5a c5b c5c; do echo -n "$v "; SI_K2_VARIANT=$v timeout 60 python tests/prof_one.py $c tc 10 kn 2>&1 | tail -1; done; done
SI_K2_VARIANT=mc4 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
