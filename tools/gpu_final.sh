set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
timeout 600 python bench.py --config 4 > gpurun_out/bench4.log 2>&1; tail -1 gpurun_out/bench4.log
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log
export BBSI_GRAPHS=0
python tools/prof_step.py --config 2 --layers 256 --energies 64 --reps 2 > gpurun_out/n_prof.log 2>&1
N=$(grep "rep 1" gpurun_out/n_prof.log | sed 's/.*, \([0-9]*\) launches/\1/')
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s $N -c $N --csv \
  python tools/prof_step.py --config 2 --layers 256 --energies 64 --reps 2 > gpurun_out/n_launches.csv 2> gpurun_out/n_launches.err
python tools/launches.py gpurun_out/n_launches.csv > gpurun_out/n_launches.txt 2>&1
python tools/launch_steps.py gpurun_out/n_launches.csv >> gpurun_out/n_launches.txt 2>&1
cat gpurun_out/n_launches.txt
