# Round-2 call K: A/B of the SM-sharing build of gj_rows_kernel (-DBBSI_GJ_SHARE_SM: 168 registers, two
# staging tiles, so a GEMM CTA of another stream group fits next to a panel CTA) against the default.
set -u
mkdir -p gpurun_out
S=paper_2605_19910_b200/_lib/libbbsi_cuda_share.so
BBSI_LIB=$S timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/k_kernels_share.log 2>&1; echo "share kernel tests rc=$?"; tail -3 gpurun_out/k_kernels_share.log
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/k_kernels.log 2>&1; echo "default kernel tests rc=$?"; tail -3 gpurun_out/k_kernels.log
for rep in 1 2; do
  for v in default share; do
    if [ $v = share ]; then export BBSI_LIB=$S; else unset BBSI_LIB; fi
    timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-traffic --steps 5 --warmup 3 > gpurun_out/k_cfg2_${v}_$rep.json 2> gpurun_out/k_cfg2_${v}_$rep.err
    python - <<PY | tee -a gpurun_out/k_ab.log
import json
r = json.load(open("gpurun_out/k_cfg2_${v}_$rep.json"))
print("$v rep $rep cfg2 ms_per_step", round(r["ms_per_step"], 2), {k: v["ms"] for k, v in r["roofline"]["kernels"].items()})
PY
  done
done
for v in default share; do
  if [ $v = share ]; then export BBSI_LIB=$S; else unset BBSI_LIB; fi
  echo "== $v" | tee -a gpurun_out/k_ab.log
  timeout 600 python bench.py --config 3 --no-e2e --no-cpu-baseline --no-traffic --steps 5 --warmup 3 > gpurun_out/k_cfg3_$v.json 2> gpurun_out/k_cfg3_$v.err
  python -c "import json; r=json.load(open('gpurun_out/k_cfg3_$v.json')); print('cfg3 ms_per_step', round(r['ms_per_step'],2))" | tee -a gpurun_out/k_ab.log
  timeout 600 python tools/bench_ddrgf.py --plans 127 127,5 --reps 2 2>&1 | grep -v "^\[" | tee -a gpurun_out/k_ab.log
  timeout 600 python tools/shard_sim.py --energies 8 16 2>&1 | tee -a gpurun_out/k_ab.log
  timeout 600 python tools/prof_step.py --config 5 --layers 128 --energies 1 --reps 3 2>&1 | tail -1 | tee -a gpurun_out/k_ab.log
done
unset BBSI_LIB
BBSI_LIB=$S timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/k_gpu_tests_share.log 2>&1; echo "share gpu tests rc=$?"; tail -3 gpurun_out/k_gpu_tests_share.log
