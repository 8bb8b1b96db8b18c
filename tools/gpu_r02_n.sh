# Round-2 call N: stream-group sweep with the SM-sharing panel (config 2 and 3).
set -u
mkdir -p gpurun_out
for g in 8 16 24 32; do
  BBSI_GROUPS=$g timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-traffic --steps 5 --warmup 3 > gpurun_out/n_cfg2_g$g.json 2> gpurun_out/n_cfg2_g$g.err
  python -c "import json; r=json.load(open('gpurun_out/n_cfg2_g$g.json')); print('cfg2 groups $g ms_per_step', round(r['ms_per_step'],2))" | tee -a gpurun_out/n_groups.log
done
for g in 8 16 32; do
  BBSI_GROUPS=$g timeout 300 python bench.py --config 3 --no-e2e --no-cpu-baseline --no-traffic --steps 5 --warmup 3 > gpurun_out/n_cfg3_g$g.json 2> gpurun_out/n_cfg3_g$g.err
  python -c "import json; r=json.load(open('gpurun_out/n_cfg3_g$g.json')); print('cfg3 groups $g ms_per_step', round(r['ms_per_step'],2))" | tee -a gpurun_out/n_groups.log
done
for g in 2 4 8; do
  echo "ddrgf groups $g" | tee -a gpurun_out/n_groups.log
  BBSI_GROUPS=$g timeout 300 python tools/bench_ddrgf.py --plans 127 127,5 --reps 2 2>&1 | grep "ddrgf plan" | tee -a gpurun_out/n_groups.log
done
