set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tuner.py tests/test_io_cli.py tests/test_gpu_dyson.py tests/test_gpu_ddrgf.py -x -q -m gpu > gpurun_out/t5_tests.log 2>&1; echo "rc=$?" >> gpurun_out/t5_tests.log
tail -3 gpurun_out/t5_tests.log
for ch in 0 32 16; do
 echo "chunk=$ch"; BBSI_E2E_TRACE=1 timeout 600 python bench.py --no-cpu-baseline --steps 2 --warmup 3 --chunk $ch > gpurun_out/t5_b$ch.log 2>&1; grep "^\[e2e\]" gpurun_out/t5_b$ch.log | tail -9; grep '^{' gpurun_out/t5_b$ch.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'])"
done 2>&1 | tee gpurun_out/t5_trace.log
