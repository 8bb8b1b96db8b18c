set -u
mkdir -p gpurun_out
for g in 1 2; do for P in 32 64; do
BBSI_GROUPS=$g timeout 600 python bench.py --config 4 --domains $P --steps 2 --warmup 3 > gpurun_out/b11_${g}_$P.log 2>&1; grep '^{' gpurun_out/b11_${g}_$P.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('groups=$g P=$P', d['ms_per_step'])"
done; done
for g in 1 2; do
BBSI_GROUPS=$g timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > gpurun_out/b11_3_$g.log 2>&1; grep '^{' gpurun_out/b11_3_$g.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 groups=$g', d['ms_per_step'])"
done
