# compute-sanitizer memcheck over the small-domain GPU parity tests
set -u
mkdir -p gpurun_out
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "bitwise_vs_oracle and (1 or 2)" > gpurun_out/san_parity.log 2>&1; echo "exit $?" >> gpurun_out/san_parity.log
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_aa.py -x -q -k "bitwise_vs_oracle or periodic or state_io" > gpurun_out/san_aa.log 2>&1; echo "exit $?" >> gpurun_out/san_aa.log
LBM_STEP_VARIANT=5 timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "bitwise_vs_oracle and tile" > gpurun_out/san_w.log 2>&1; echo "exit $?" >> gpurun_out/san_w.log
