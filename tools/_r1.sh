cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo "bench rc=$?" >> gpurun_out/bench_r2b.err
timeout 900 python tools/dense_vs_sparse.py > gpurun_out/dense_vs_sparse_r2.md 2> gpurun_out/dense_vs_sparse_r2.err
