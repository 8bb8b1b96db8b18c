# Round-2 evidence on one B200: the bench line of every configuration (roofline with the
# ncu DRAM-traffic probe, CPU baseline, e2e), the reference arm, the launch list of one
# config-2 solve and ncu --set full captures of the top kernels.
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/r02_bench_cfg2.json 2> gpurun_out/r02_bench_cfg2.err; echo "cfg2 rc=$?"
python bench.py --config 3 > gpurun_out/r02_bench_cfg3.json 2> gpurun_out/r02_bench_cfg3.err; echo "cfg3 rc=$?"
python bench.py --config 4 > gpurun_out/r02_bench_cfg4.json 2> gpurun_out/r02_bench_cfg4.err; echo "cfg4 rc=$?"
python bench.py --config 5 --steps 1 --warmup 3 > gpurun_out/r02_bench_cfg5.json 2> gpurun_out/r02_bench_cfg5.err; echo "cfg5 rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err; echo "ref rc=$?"
export BBSI_GRAPHS=0
python tools/prof_step.py --config 2 --layers 256 --energies 64 --reps 2 > gpurun_out/r02_prof.log 2>&1
N=$(grep "rep 1" gpurun_out/r02_prof.log | sed 's/.*, \([0-9]*\) launches/\1/')
echo "launches per solve: $N"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s $N -c $N --csv \
  python tools/prof_step.py --config 2 --layers 256 --energies 64 --reps 2 > gpurun_out/r02_launches.csv 2> gpurun_out/r02_launches.err
python tools/launches.py gpurun_out/r02_launches.csv > gpurun_out/r02_launches.txt 2>&1
for spec in "zgemm_tma_kernel 40 sweep_tma" "zgemm_grouped_kernel 203 gjgemm" "gj_pair_kernel 203 pair"; do
  set -- $spec
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$1" -s $2 -c 1 -o gpurun_out/r02_full_$3 \
    python tools/prof_step.py --config 2 --layers 128 --energies 64 --reps 1 > gpurun_out/r02_full_$3.log 2>&1
  echo "$3 rc=$?"
done
