# 2-GPU suite: configs[2] at 2 stages (k sweep) and the square-wave trace.
B="timeout -k 10 420 python bench.py --gpus 2 --no-cpu-baseline"
$B --steps 10 --warmup 3 --k-sweep > gpurun_out/${PFX:-r2f}_n2_c3.json 2> gpurun_out/${PFX:-r2f}_n2_c3.err; echo c3 rc=$?
$B --steps 20 --warmup 3 --k-sweep --trace square --period-ms 1200 --link-gbps 400 --availability 0.1 --retune 2 --passive-profile --tuner-repeats 1 > gpurun_out/${PFX:-r2f}_n2_square.json 2> gpurun_out/${PFX:-r2f}_n2_square.err; echo square rc=$?
python scripts/bench_summary.py gpurun_out/${PFX:-r2f}_n2_*.json
