# Round-2 call C: gj_rows_kernel after the pair-step fix: tests, clock64 phase marks, A/B timings.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/c_kernels.log 2>&1; echo "kernel tests rc=$?"; tail -4 gpurun_out/c_kernels.log
for cfg in "256 128" "256 2" "128 64" "512 16" "768 2"; do
  set -- $cfg
  BBSI_LIB=paper_2605_19910_b200/_lib/libbbsi_cuda_dbg.so timeout 300 python tools/dbg_zinv_rows.py --block $1 --batch $2 2>&1 | tail -1 | tee -a gpurun_out/c_marks.log
done
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/c_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -5 gpurun_out/c_gpu_tests.log
for m in 4 0; do
  export BBSI_GJ_ROWS=$m
  echo "=== BBSI_GJ_ROWS=$m" | tee -a gpurun_out/c_ab.log
  timeout 600 python tools/bench_ddrgf.py --plans 127 127,5 --reps 2 2>&1 | grep -v "^\[" | tee -a gpurun_out/c_ab.log
  timeout 600 python tools/prof_step.py --config 5 --layers 128 --energies 1 --reps 3 2>&1 | tee -a gpurun_out/c_ab.log
  timeout 600 python tools/shard_sim.py --energies 8 16 2>&1 | tee -a gpurun_out/c_ab.log
done
unset BBSI_GJ_ROWS
