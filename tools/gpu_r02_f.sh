# Round-2 call F: full-size parity of configs 4, 3, 2, 1 against the compiled reference (every energy).
set -u
mkdir -p gpurun_out
PARITY_CONFIGS="4 3 2 1" PARITY_TIMEOUT=3000 bash tools/gpu_parity.sh
