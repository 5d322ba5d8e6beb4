# One-GPU round check: every -m gpu test, smoke(), the attention microbenchmark and the N=1 bench.
timeout -k 10 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 --timeout-method thread -x > gpurun_out/r2_gpu_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2_gpu_tests.log
timeout -k 5 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -k 5 120 python scripts/bench_attention.py > gpurun_out/r2_attn.log 2>&1; cat gpurun_out/r2_attn.log
timeout -k 10 400 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_n1.json 2> gpurun_out/r2_bench_n1.err; echo bench rc=$?; python scripts/bench_summary.py gpurun_out/r2_bench_n1.json
