# ncu evidence for the current code: launch list of one full config-2 solve (BBSI_GRAPHS=0,
# eager launches, second rep) and --set full captures of the three top kernels.
# Launch order inside one stream group's inward step: 8 x (pair panel, GJ GEMM), lm GEMM
# (1024 tiles), window+um GEMM (2048 tiles): zgemm launch 209 = a window+um GEMM,
# zgemm launch 203 / pair launch 203 = GJ step 3 of an inversion.
set -u
mkdir -p gpurun_out
export BBSI_GRAPHS=0
python tools/prof_step.py --config 2 --layers 256 --energies 64 --reps 2 > gpurun_out/n_prof.log 2>&1
N=$(grep "rep 1" gpurun_out/n_prof.log | sed 's/.*, \([0-9]*\) launches/\1/')
echo "launches per solve: $N"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s $N -c $N --csv \
  python tools/prof_step.py --config 2 --layers 256 --energies 64 --reps 2 > gpurun_out/n_launches.csv 2> gpurun_out/n_launches.err
python tools/launches.py gpurun_out/n_launches.csv > gpurun_out/n_launches.txt 2>&1
python tools/launch_steps.py gpurun_out/n_launches.csv >> gpurun_out/n_launches.txt 2>&1
cat gpurun_out/n_launches.txt
for spec in "zgemm_grouped_kernel 209 sweep" "zgemm_grouped_kernel 203 gjgemm" "gj_pair_kernel 203 pair"; do
  set -- $spec
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$1" -s $2 -c 1 -o gpurun_out/n_full_$3 \
    python tools/prof_step.py --config 2 --layers 128 --energies 64 --reps 1 > gpurun_out/n_full_$3.log 2>&1
  echo "$3 rc=$?"
done
