# ncu evidence for the current code: launch list of one full config-2 solve (BBSI_GRAPHS=0,
# eager launches, second rep) and --set full captures of the three top kernels.
set -u
mkdir -p gpurun_out
export BBSI_GRAPHS=0
python tools/prof_step.py --config 2 --layers 256 --energies 64 --reps 2 > gpurun_out/n_prof.log 2>&1
cat gpurun_out/n_prof.log
N=$(grep "rep 1" gpurun_out/n_prof.log | sed 's/.*, \([0-9]*\) launches/\1/')
echo "launches per solve: $N"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s $N -c $N --csv \
  python tools/prof_step.py --config 2 --layers 256 --energies 64 --reps 2 > gpurun_out/n_launches.csv 2> gpurun_out/n_launches.err
python tools/launches.py gpurun_out/n_launches.csv > gpurun_out/n_launches.txt 2>&1; head -20 gpurun_out/n_launches.txt
# full sections of one sweep GEMM (4096 tiles), one GJ GEMM, one pair panel, at layer ~60 of a 128-layer solve
for k in "zgemm_grouped_kernel<0" "zgemm_grouped_kernel<1" "gj_pair_kernel"; do
  tag=$(echo "$k" | tr -c 'a-z0-9' '_')
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$k" -s 200 -c 1 -o gpurun_out/n_full_$tag \
    python tools/prof_step.py --config 2 --layers 128 --energies 64 --reps 1 > gpurun_out/n_full_$tag.log 2>&1
  echo "$k rc=$?"
done
ls -la gpurun_out/
