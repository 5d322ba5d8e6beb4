# The round-end driver's command forms on one GPU: pytest -m gpu, smoke(), an ncu launch capture of
# smoke(), the bench's reference arm and our arm (N=1, 20 steps, 5 warm-up).
timeout -k 10 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 --timeout-method thread > gpurun_out/${PFX:-r2_final}_gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${PFX:-r2_final}_gpu_tests.log
timeout -k 5 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${PFX:-r2_final}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${PFX:-r2_final}_smoke.log
timeout -k 10 700 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/${PFX:-r2_final}_launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${PFX:-r2_final}_ncu_smoke.log 2>&1; echo "ncu smoke rc=$?"
timeout -k 10 900 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${PFX:-r2_final}_ref1.json 2> gpurun_out/${PFX:-r2_final}_ref1.err; echo "ref rc=$?"; tail -c 300 gpurun_out/${PFX:-r2_final}_ref1.json
timeout -k 10 600 python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${PFX:-r2_final}_n1.json 2> gpurun_out/${PFX:-r2_final}_n1.err; echo "bench rc=$?"; python scripts/bench_summary.py gpurun_out/${PFX:-r2_final}_n1.json
