# compute-sanitizer racecheck / synccheck over the shared-memory tile kernels
set -u
mkdir -p gpurun_out
timeout 1800 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "bitwise_vs_oracle and tile and 1" > gpurun_out/san_race.log 2>&1; echo "exit $?" >> gpurun_out/san_race.log
LBM_STEP_VARIANT=6 timeout 1800 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "bitwise_vs_oracle and tile and 1" > gpurun_out/san_race6.log 2>&1; echo "exit $?" >> gpurun_out/san_race6.log
timeout 1800 compute-sanitizer --tool synccheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_aa.py -x -q -k "bitwise_vs_oracle and 1" > gpurun_out/san_sync.log 2>&1; echo "exit $?" >> gpurun_out/san_sync.log
