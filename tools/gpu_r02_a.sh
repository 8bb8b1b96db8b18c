# Round-2 call A: config-5 full-size parity (streaming oracle, 8 energies, GPU RGF + DDRGF),
# the config-5 bench line, then the GPU suite.
set -u
mkdir -p gpurun_out
nproc > gpurun_out/r02_parity_host.txt; free -g >> gpurun_out/r02_parity_host.txt
PARITY_CONFIGS="5" PARITY_TIMEOUT=4500 bash tools/gpu_parity.sh
timeout 1500 python bench.py --config 5 --steps 1 --warmup 3 > gpurun_out/r02_bench_cfg5.json 2> gpurun_out/r02_bench_cfg5.err; echo "cfg5 rc=$?"
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r02_gpu_tests.log
