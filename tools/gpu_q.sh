cd /root/repo
timeout 1500 compute-sanitizer --tool initcheck --print-limit 10 python -m pytest -q -x -m gpu \
    "tests/test_refine.py::test_large_cuts_equal_oracle[0]" "tests/test_delta.py::test_caller_delta_unordered_with_stale_duplicates[0]" "tests/test_delta.py::test_sync_repacks_and_relocates" "tests/test_prefetch_round.py::test_prefetch_round_equals_reference_loop[3]" > gpurun_out/san_initcheck.log 2>&1
echo "initcheck rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/san_initcheck.log | tail -2 | tr '\n' ' ')"
grep -A6 "Uninitialized" gpurun_out/san_initcheck.log | head -16
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
