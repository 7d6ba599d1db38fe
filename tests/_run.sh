SI_K2T_TRACE=/tmp/t.bin timeout 60 python tests/prof_one.py c5b tc 1 nk 2>&1 | tail -1; python tools/k2t_trace.py /tmp/t.bin | tail -14
