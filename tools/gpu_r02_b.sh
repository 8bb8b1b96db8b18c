# Round-2 call B: gj_rows_kernel (register-resident Gauss-Jordan panels, clusters for n > 256):
# kernel tests, the GPU suite, then A/B timings against the LU + Pinv panels (BBSI_GJ_ROWS=0).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/b_kernels.log 2>&1; echo "kernel tests rc=$?"; tail -15 gpurun_out/b_kernels.log
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/b_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -5 gpurun_out/b_gpu_tests.log
for m in 4 0; do
  export BBSI_GJ_ROWS=$m
  echo "=== BBSI_GJ_ROWS=$m" | tee -a gpurun_out/b_ab.log
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-traffic --steps 3 --warmup 3 > gpurun_out/b_cfg2_rows$m.json 2> gpurun_out/b_cfg2_rows$m.err; echo "cfg2 rc=$?"
  python - <<PY | tee -a gpurun_out/b_ab.log
import json
try:
    r = json.load(open("gpurun_out/b_cfg2_rows$m.json"))
    print("cfg2 ms_per_step", r["ms_per_step"], {k: (v["ms"], v["tflops"]) for k, v in r["roofline"]["kernels"].items()})
except Exception as ex:
    print("cfg2 parse failed", ex)
PY
  timeout 600 python bench.py --config 3 --no-e2e --no-cpu-baseline --no-traffic --steps 3 --warmup 3 > gpurun_out/b_cfg3_rows$m.json 2> gpurun_out/b_cfg3_rows$m.err; echo "cfg3 rc=$?"
  python - <<PY | tee -a gpurun_out/b_ab.log
import json
try:
    r = json.load(open("gpurun_out/b_cfg3_rows$m.json"))
    print("cfg3 ms_per_step", r["ms_per_step"], {k: (v["ms"], v["tflops"]) for k, v in r["roofline"]["kernels"].items()})
except Exception as ex:
    print("cfg3 parse failed", ex)
PY
  timeout 600 python tools/bench_ddrgf.py --plans 127 127,5 --reps 2 2>&1 | grep -v "^\[" | tee -a gpurun_out/b_ab.log
  timeout 600 python tools/prof_step.py --config 5 --layers 128 --energies 1 --reps 3 2>&1 | tee -a gpurun_out/b_ab.log
  timeout 600 python tools/shard_sim.py --energies 8 16 2>&1 | tee -a gpurun_out/b_ab.log
done
unset BBSI_GJ_ROWS
for g in 4 8; do
  echo "=== rows default, BBSI_GROUPS=$g (ddrgf)" | tee -a gpurun_out/b_ab.log
  BBSI_GROUPS=$g timeout 600 python tools/bench_ddrgf.py --plans 127,5 --reps 2 2>&1 | grep -v "^\[" | tee -a gpurun_out/b_ab.log
done
