set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_io_cli.py tests/test_gpu_dyson.py -x -q -m gpu > gpurun_out/t3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/t3_tests.log
tail -3 gpurun_out/t3_tests.log
for ch in 0 32 16; do
 echo "chunk=$ch"; timeout 600 python bench.py --no-cpu-baseline --steps 2 --warmup 3 --chunk $ch 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e'])"
done 2>&1 | tee gpurun_out/t3_e2e.log
