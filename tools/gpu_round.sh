#!/bin/bash
# One GPU call: tests, smoke, bench, reference arm, PCIe ceiling, ncu launch
# list, ncu full captures of the dominant kernel (K2, config 5b, token-major)
# and of the 2:4 kernels K3 and K4 on the same linear (per-variant table).  Each ncu
# step runs only after the same command exited 0 without ncu.
set -u
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python tools/pcie_bw.py > gpurun_out/pcie_bw.txt 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 --no-secondary"
if timeout 600 $CMD > gpurun_out/plain_launch.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
     --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
fi
for V in "top tc k2p" "sp sp k3" "ws ws k4"; do
  set -- $V
  P1="python tests/prof_one.py c5b $2 3 nk"
  if timeout 300 $P1 > gpurun_out/plain_prof_$1.log 2>&1; then
    rm -f /tmp/prof_$1.ncu-rep
    timeout 900 ncu -f --set full --clock-control none -k regex:$3 -s 2 -c 1 \
       -o /tmp/prof_$1 $P1 > gpurun_out/ncu_full_$1.log 2>&1
    ncu -i /tmp/prof_$1.ncu-rep --page raw --csv > gpurun_out/prof_$1_raw.csv 2>/dev/null
    ncu -i /tmp/prof_$1.ncu-rep --page details --csv > gpurun_out/prof_$1_details.csv 2>/dev/null
  fi
done
echo done
