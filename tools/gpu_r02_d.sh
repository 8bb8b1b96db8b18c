# Round-2 call D: gj_rows_kernel with shared-memory operands in the tails and coalesced V output.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/d_kernels.log 2>&1; echo "kernel tests rc=$?"; tail -4 gpurun_out/d_kernels.log
for cfg in "256 128" "256 2" "128 64" "512 16" "768 2"; do
  set -- $cfg
  BBSI_LIB=paper_2605_19910_b200/_lib/libbbsi_cuda_dbg.so timeout 300 python tools/dbg_zinv_rows.py --block $1 --batch $2 2>&1 | tail -1 | tee -a gpurun_out/d_marks.log
done
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-traffic --steps 3 --warmup 3 > gpurun_out/d_cfg2.json 2> gpurun_out/d_cfg2.err; echo "cfg2 rc=$?"
timeout 600 python bench.py --config 3 --no-e2e --no-cpu-baseline --no-traffic --steps 3 --warmup 3 > gpurun_out/d_cfg3.json 2> gpurun_out/d_cfg3.err; echo "cfg3 rc=$?"
python - <<PY | tee -a gpurun_out/d_ab.log
import json
for f in ("d_cfg2", "d_cfg3"):
    try:
        r = json.load(open(f"gpurun_out/{f}.json"))
        print(f, "ms_per_step", r["ms_per_step"], {k: (v["ms"], v["tflops"]) for k, v in r["roofline"]["kernels"].items()})
    except Exception as ex:
        print(f, "parse failed", ex)
PY
timeout 600 python tools/bench_ddrgf.py --plans 127 127,5 --reps 2 2>&1 | grep -v "^\[" | tee -a gpurun_out/d_ab.log
timeout 600 python tools/prof_step.py --config 5 --layers 128 --energies 1 --reps 3 2>&1 | tee -a gpurun_out/d_ab.log
timeout 600 python tools/shard_sim.py --energies 8 16 2>&1 | tee -a gpurun_out/d_ab.log
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/d_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -5 gpurun_out/d_gpu_tests.log
