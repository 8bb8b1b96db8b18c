set -u
mkdir -p gpurun_out
timeout 2400 python bench.py --config 5 --steps 1 --warmup 3 > gpurun_out/r02_bench_cfg5.json 2> gpurun_out/r02_bench_cfg5.err; echo "cfg5 rc=$?"
PARITY_TIMEOUT=6000 bash tools/gpu_parity.sh
