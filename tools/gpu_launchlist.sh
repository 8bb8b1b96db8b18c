set -u
mkdir -p gpurun_out
export BBSI_GRAPHS=0
python tools/prof_step.py --config 2 --layers 64 --energies 64 --reps 2 > gpurun_out/l_prof.log 2>&1
N=$(grep "rep 1" gpurun_out/l_prof.log | sed 's/.*, \([0-9]*\) launches/\1/')
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s $N -c $N --csv \
  python tools/prof_step.py --config 2 --layers 64 --energies 64 --reps 2 > gpurun_out/l_launches.csv 2> gpurun_out/l_launches.err
python tools/launches.py gpurun_out/l_launches.csv | head -12
