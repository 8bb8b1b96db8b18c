# Split pair panel (several CTAs per matrix for small batches) and DDRGF stream groups:
# kernel tests, full GPU suite, then A/B timings on one B200.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/split_kernels.log 2>&1; echo "kernel tests rc=$?"; tail -2 gpurun_out/split_kernels.log
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/split_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/split_gpu_tests.log
echo "default split, groups 2: plans" >> gpurun_out/split_ddrgf.log
BBSI_DDRGF_TRACE=1 timeout 900 python tools/bench_ddrgf.py --plans 127 127,3 127,5 127,7 127,5,2 63,7 63,5,3 --reps 2 >> gpurun_out/split_ddrgf.log 2>&1
for sp in 1 0; do
  for g in 1 4 8; do
    if [ $sp = 1 ]; then export BBSI_PANEL_SPLIT=1; else unset BBSI_PANEL_SPLIT; fi
    echo "split=$sp groups=$g" >> gpurun_out/split_ddrgf.log
    BBSI_GROUPS=$g timeout 600 python tools/bench_ddrgf.py --plans 127,5 --reps 2 >> gpurun_out/split_ddrgf.log 2>&1
  done
done
unset BBSI_PANEL_SPLIT
for sp in 1 0; do
  if [ $sp = 1 ]; then export BBSI_PANEL_SPLIT=1; else unset BBSI_PANEL_SPLIT; fi
  echo "split=$sp" >> gpurun_out/split_shards.log
  timeout 600 python tools/shard_sim.py --energies 64 32 16 8 >> gpurun_out/split_shards.log 2>&1
done
unset BBSI_PANEL_SPLIT
grep -v "^\[" gpurun_out/split_ddrgf.log; cat gpurun_out/split_shards.log
