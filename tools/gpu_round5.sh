set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1
grep '^{' gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'], {k:(v['launches'],round(v['ms'],1)) for k,v in d['roofline']['kernels'].items()})"
timeout 600 python bench.py --config 4 --steps 2 --warmup 3 > gpurun_out/bench4.log 2>&1; tail -1 gpurun_out/bench4.log
bash tools/gpu_launchlist.sh > /dev/null 2>&1; python tools/launch_steps.py gpurun_out/l_launches.csv
