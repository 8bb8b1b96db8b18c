# Round-2 evidence on one B200: the bench line of every configuration (roofline with the
# ncu DRAM-traffic probe, CPU baseline, e2e), the reference arm, and ncu --set full
# captures of the top kernels at full occupancy (one stream group: 2048-tile launches).
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/r02_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r02_gpu_tests.log
BBSI_GJ_ROWS=0 python bench.py --no-e2e --no-cpu-baseline --no-traffic > gpurun_out/r02_cfg2_lu_panels.json 2> gpurun_out/r02_cfg2_lu_panels.err; echo "lu panels rc=$?"
python bench.py > gpurun_out/r02_bench_cfg2.json 2> gpurun_out/r02_bench_cfg2.err; echo "cfg2 rc=$?"
python bench.py --config 3 > gpurun_out/r02_bench_cfg3.json 2> gpurun_out/r02_bench_cfg3.err; echo "cfg3 rc=$?"
python bench.py --config 4 > gpurun_out/r02_bench_cfg4.json 2> gpurun_out/r02_bench_cfg4.err; echo "cfg4 rc=$?"
BBSI_DDRGF_TRACE=1 timeout 900 python tools/bench_ddrgf.py --plans 127 127,5 255 63,7 --reps 2 > gpurun_out/r02_ddrgf_plans.log 2>&1; echo "plans rc=$?"
timeout 1800 python bench.py --config 5 --steps 1 --warmup 3 > gpurun_out/r02_bench_cfg5.json 2> gpurun_out/r02_bench_cfg5.err; echo "cfg5 rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err; echo "ref rc=$?"
export BBSI_GRAPHS=0 BBSI_GROUPS=1
for spec in "zgemm_tma_kernel 6 2 sweep_tma" "zgemm_grouped_kernel 24 1 gjgemm" "gj_rows_kernel 24 1 gjrows"; do
  set -- $spec
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$1" -s $2 -c $3 -o gpurun_out/r02_full_$4 \
    python tools/prof_step.py --config 2 --layers 64 --energies 64 --reps 1 > gpurun_out/r02_full_$4.log 2>&1
  echo "$4 rc=$?"
done
unset BBSI_GROUPS
# ncu launch list of ONE full config-2 solve (eager launches, default stream groups; second rep)
python tools/prof_step.py --config 2 --layers 256 --energies 64 --reps 2 > gpurun_out/r02_prof.log 2>&1
N=$(grep "rep 1" gpurun_out/r02_prof.log | sed 's/.*, \([0-9]*\) launches/\1/')
echo "launches per solve: $N"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s $N -c $N --csv \
  python tools/prof_step.py --config 2 --layers 256 --energies 64 --reps 2 > gpurun_out/r02_launches_step.csv 2> gpurun_out/r02_launches.err
python tools/launches.py gpurun_out/r02_launches_step.csv > gpurun_out/r02_launches_step.txt 2>&1
python tools/launch_steps.py gpurun_out/r02_launches_step.csv >> gpurun_out/r02_launches_step.txt 2>&1
gzip -f gpurun_out/r02_launches_step.csv
cat gpurun_out/r02_launches_step.txt | head -30
