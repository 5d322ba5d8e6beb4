# compute-sanitizer over small cases of every kernel family and the executor's flag protocol.
# One tool per gpurun call (B200_PROFILING.md); usage: bash scripts/sanitize.sh memcheck|racecheck|synccheck
tool=$1
sel="tests/test_gemm_gpu.py::test_gemm_epilogues tests/test_gemm_gpu.py::test_gemm_pair_epilogues_and_wgrad tests/test_gemm_gpu.py::test_gemm_two_k_segments tests/test_attention_gpu.py::test_flash_forward tests/test_attention_gpu.py::test_flash_backward tests/test_stage_gpu.py::test_toy_single_stage_matches_oracle tests/test_pipeline_gpu.py::test_plan_that_cannot_merge_raises_deadlock tests/test_stage_gpu.py::test_two_stages_one_process_one_gpu"
k="not 1024-32 and not 8-1024 and not 16-512 and not 4-1024"
timeout -k 10 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 --target-processes all \
    python -m pytest $sel -k "$k" -q -p no:cacheprovider -x > gpurun_out/r2_sanitizer_$tool.log 2>&1
echo "$tool rc=$?" | tee -a gpurun_out/r2_sanitizer_$tool.log
grep -E "ERROR SUMMARY|passed|failed|Error" gpurun_out/r2_sanitizer_$tool.log | tail -5
