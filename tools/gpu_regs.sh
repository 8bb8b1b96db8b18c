set -u
mkdir -p gpurun_out
run() { echo "$*"; env "$@" timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('   ', d['ms_per_step'], {k:(v['launches'],round(v['ms'],1)) for k,v in d['roofline']['kernels'].items()})"; }
{
run BBSI_PAIR_PRE2=1
run BBSI_LIB=$PWD/paper_2605_19910_b200/_lib/libbbsi_cuda_r168.so BBSI_PAIR_PRE2=1
run BBSI_LIB=$PWD/paper_2605_19910_b200/_lib/libbbsi_cuda_r168.so BBSI_PAIR_PRE2=0
run BBSI_PAIR_PRE2=0
} 2>&1 | tee gpurun_out/regs.log
