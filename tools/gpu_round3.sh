set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_rgf.py tests/test_gpu_dyson.py -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1
grep '^{' gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'], {k:(v['launches'],round(v['ms'],1)) for k,v in d['roofline']['kernels'].items()})"
bash tools/gpu_launchlist.sh > /dev/null 2>&1; python tools/launch_steps.py gpurun_out/l_launches.csv | head -2
timeout 900 python tools/bench_ddrgf.py --config 4 --domains 8 16 32 64 > gpurun_out/ddrgf4.log 2>&1; cat gpurun_out/ddrgf4.log
timeout 900 python tools/bench_ddrgf.py --config 5 --layers 256 --domains 4 8 > gpurun_out/ddrgf5.log 2>&1; cat gpurun_out/ddrgf5.log
