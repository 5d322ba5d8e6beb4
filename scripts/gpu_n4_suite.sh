# 4-GPU suite: configs[2] (GPT-1.3B, constant 50 % at 100 Gb/s, k sweep), configs[4] (BERT-large bursty),
# configs[3] at 4 stages (GPT-6.7B under a 60 GB cap, two-regime trace), and the square-wave trace.
B="timeout -k 10 420 python bench.py --gpus 4 --no-cpu-baseline"
$B --steps 10 --warmup 3 --k-sweep > gpurun_out/${PFX:-r2f}_n4_c3.json 2> gpurun_out/${PFX:-r2f}_n4_c3.err; echo c3 rc=$?
$B --model bert-large --global-batch 64 --micro-batch 4 --steps 10 --warmup 3 --k-sweep --trace bursty --on-ms 150 --off-ms 150 --retune 2 --passive-profile --tuner-repeats 1 > gpurun_out/${PFX:-r2f}_n4_bert_bursty.json 2> gpurun_out/${PFX:-r2f}_n4_bert_bursty.err; echo bert rc=$?
$B --model 6.7b --global-batch 64 --micro-batch 1 --mem-cap-gb 60 --steps 6 --warmup 3 --k-sweep --trace two-regime --availability 0.3 --regime-ms 2500 --retune 2 --passive-profile --tuner-repeats 1 > gpurun_out/${PFX:-r2f}_n4_67b_cap.json 2> gpurun_out/${PFX:-r2f}_n4_67b_cap.err; echo 67b rc=$?
$B --steps 30 --warmup 3 --k-sweep --trace square --period-ms 1200 --link-gbps 400 --availability 0.1 --retune 2 --passive-profile --tuner-repeats 1 > gpurun_out/${PFX:-r2f}_n4_square.json 2> gpurun_out/${PFX:-r2f}_n4_square.err; echo square rc=$?
python scripts/bench_summary.py gpurun_out/${PFX:-r2f}_n4_*.json; grep -m2 "nRanks" gpurun_out/${PFX:-r2f}_n4_c3.err
