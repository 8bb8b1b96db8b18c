set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_rgf.py tests/test_gpu_dyson.py tests/test_gpu_ddrgf.py -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
for c in 1 0; do
BBSI_GJ_CLATE=$c timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/bench_c$c.log 2>&1
grep '^{' gpurun_out/bench_c$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('clate=$c', d['ms_per_step'], {k:(v['launches'],round(v['ms'],1)) for k,v in d['roofline']['kernels'].items()})"
done
bash tools/gpu_launchlist.sh > /dev/null 2>&1; python tools/launch_steps.py gpurun_out/l_launches.csv
