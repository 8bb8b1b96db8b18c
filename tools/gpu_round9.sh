set -u
mkdir -p gpurun_out
for v in 2 3; do
BBSI_GJ_MINB=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/b9_$v.log 2>&1
grep '^{' gpurun_out/b9_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gj_minb=$v', d['ms_per_step'], {k:(v['launches'],round(v['ms'],1)) for k,v in d['roofline']['kernels'].items()})"
done
