set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dyson.py tests/test_gpu_rgf.py -x -q -m gpu > gpurun_out/gpu_tests10.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests10.log
tail -3 gpurun_out/gpu_tests10.log
for f in 1 0; do
BBSI_FORM_IN_GEMM=$f timeout 600 python bench.py --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/b10_$f.log 2>&1
grep '^{' gpurun_out/b10_$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('form_in_gemm=$f', d['ms_per_step'], d['e2e']['ms_per_step'], {k:(v['launches'],round(v['ms'],1)) for k,v in d['roofline']['kernels'].items()})"
done
