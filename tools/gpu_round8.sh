set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dyson.py -x -q -m gpu > gpurun_out/gpu_tests8.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests8.log
tail -3 gpurun_out/gpu_tests8.log
timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > gpurun_out/bench3.log 2>&1
grep '^{' gpurun_out/bench3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', d['ms_per_step'], d['tflops_algorithmic'])"
timeout 1200 python -u tools/parity_full.py --configs 3 > gpurun_out/parity3_dense.log 2>&1; cat gpurun_out/parity3_dense.log
