set -u
mkdir -p gpurun_out
for ch in 16 20 22 28; do
 timeout 600 python bench.py --no-cpu-baseline --steps 2 --warmup 3 --chunk $ch > gpurun_out/b7_$ch.log 2>&1; grep '^{' gpurun_out/b7_$ch.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunk=$ch', d['ms_per_step'], d['e2e']['ms_per_step'])"
done
timeout 1200 python -u tools/parity_full.py --configs 3 > gpurun_out/parity3.log 2>&1; cat gpurun_out/parity3.log
for P in 16 24 48; do timeout 600 python bench.py --config 4 --domains $P --steps 2 --warmup 3 > gpurun_out/b7_4_$P.log 2>&1; grep '^{' gpurun_out/b7_4_$P.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 P=$P', d['ms_per_step'])"; done
