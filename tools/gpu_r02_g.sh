# Round-2 call G: gj_rows_kernel with the pull-based cluster exchange and the M2 prefetch:
# tests, phase marks, A/B timings of the latency-bound workloads.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/g_kernels.log 2>&1; echo "kernel tests rc=$?"; tail -4 gpurun_out/g_kernels.log
for lib in libbbsi_cuda_dbg.so libbbsi_cuda_dbg2.so; do
  echo "== $lib" | tee -a gpurun_out/g_marks.log
  for cfg in "256 128" "256 2" "128 64" "512 16" "768 2" "1024 2"; do
    set -- $cfg
    BBSI_LIB=paper_2605_19910_b200/_lib/$lib timeout 300 python tools/dbg_zinv_rows.py --block $1 --batch $2 2>&1 | tail -1 | tee -a gpurun_out/g_marks.log
  done
done
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/g_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -5 gpurun_out/g_gpu_tests.log
timeout 600 python tools/bench_ddrgf.py --plans 127 127,5 --reps 2 2>&1 | grep -v "^\[" | tee -a gpurun_out/g_ab.log
timeout 600 python tools/prof_step.py --config 5 --layers 128 --energies 1 --reps 3 2>&1 | tee -a gpurun_out/g_ab.log
timeout 600 python tools/shard_sim.py --energies 8 16 2>&1 | tee -a gpurun_out/g_ab.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-traffic --steps 3 --warmup 3 > gpurun_out/g_cfg2.json 2> gpurun_out/g_cfg2.err; echo "cfg2 rc=$?"
python - <<PY | tee -a gpurun_out/g_ab.log
import json
r = json.load(open("gpurun_out/g_cfg2.json"))
print("cfg2 ms_per_step", r["ms_per_step"], {k: (v["ms"], v["tflops"]) for k, v in r["roofline"]["kernels"].items()})
PY
