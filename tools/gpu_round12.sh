set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dyson.py -x -q -m gpu > gpurun_out/gpu_tests12.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests12.log
tail -2 gpurun_out/gpu_tests12.log
for f in 1 0; do
BBSI_GJ_PERSIST=$f timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/b12_$f.log 2>&1
grep '^{' gpurun_out/b12_$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('persist=$f', d['ms_per_step'], {k:(v['launches'],round(v['ms'],1)) for k,v in d['roofline']['kernels'].items()})"
done
