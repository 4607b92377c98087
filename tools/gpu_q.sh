cd /root/repo
O=gpurun_out/san; mkdir -p $O
timeout 1500 compute-sanitizer --tool initcheck --print-limit 5 python -m pytest -q -x -m gpu "tests/test_shard.py::test_interval_sums_bound" "tests/test_gpu_parity.py::test_ctx_wait_stream_orders_device_inputs" "tests/test_prefetch_round.py::test_prefetch_round_equals_reference_loop[7]" "tests/test_refine.py::test_device_sort_fallback_equals_oracle[0]" > $O/final_initcheck.log 2>&1
echo "initcheck rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' $O/final_initcheck.log | tail -2 | tr '\n' ' ')"
grep -A4 "Uninitialized" $O/final_initcheck.log | head -12
