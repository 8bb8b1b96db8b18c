set -u
mkdir -p gpurun_out
run() { echo "$*"; env "$@" timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('   ', d['ms_per_step'])"; }
{
run BBSI_GROUPS=2
run BBSI_GROUPS=3
run BBSI_GROUPS=4
run BBSI_GROUPS=2 BBSI_PANEL_PRIORITY=0
run BBSI_GROUPS=2 BBSI_GEMM_MINB=2
run BBSI_GROUPS=1 BBSI_GEMM_MINB=2
} 2>&1 | tee gpurun_out/t6_env.log
