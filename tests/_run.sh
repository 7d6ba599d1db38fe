export SI_K2_VARIANT=tmemw
for d in 0 1 16 17 8193 8209; do echo -n "tmemw debug=$d "; SI_K2_DEBUG=$d timeout 60 python tests/prof_one.py c5b tc 10 nk 2>&1 | tail -1; done
