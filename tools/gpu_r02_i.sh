# Round-2 call I: GPU suite on the final library, config-4 bench line + DDRGF plans, then the
# config-5 full-size parity pass (8 energies, GPU RGF + DDRGF with the cluster panels).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r02_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r02_gpu_tests.log
timeout 400 python bench.py --config 4 > gpurun_out/r02_bench_cfg4.json 2> gpurun_out/r02_bench_cfg4.err; echo "cfg4 rc=$?"
BBSI_DDRGF_TRACE=1 timeout 300 python tools/bench_ddrgf.py --plans 127 127,5 255 63,7 --reps 2 > gpurun_out/r02_ddrgf_plans.log 2>&1; echo "plans rc=$?"
PARITY_CONFIGS="5" PARITY_TIMEOUT=3050 bash tools/gpu_parity.sh
