set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dyson.py tests/test_gpu_ddrgf.py tests/test_gpu_rgf.py -x -q -m gpu > gpurun_out/gpu_tests6.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests6.log
tail -3 gpurun_out/gpu_tests6.log
for te in 1 0; do
BBSI_TWO_ENDED=$te timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > gpurun_out/bench3_$te.log 2>&1
grep '^{' gpurun_out/bench3_$te.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 two_ended=$te', d['ms_per_step'], d['tflops_algorithmic'])"
done
timeout 600 python bench.py --config 4 --steps 2 --warmup 3 > gpurun_out/bench4.log 2>&1; grep '^{' gpurun_out/bench4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 P=32', d['ms_per_step'])"
timeout 600 python bench.py --config 4 --domains 64 --steps 2 --warmup 3 > gpurun_out/bench4b.log 2>&1; grep '^{' gpurun_out/bench4b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 P=64', d['ms_per_step'])"
for ch in 24 40; do
 timeout 600 python bench.py --no-cpu-baseline --steps 2 --warmup 3 --chunk $ch > gpurun_out/b6_$ch.log 2>&1; grep '^{' gpurun_out/b6_$ch.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunk=$ch', d['ms_per_step'], d['e2e']['ms_per_step'])"
done
