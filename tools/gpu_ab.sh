set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dyson.py -x -q > gpurun_out/t2_dyson.log 2>&1; echo "rc=$?" >> gpurun_out/t2_dyson.log
tail -5 gpurun_out/t2_dyson.log
for te in 1 0; do for g in 1 2; do
 echo "two_ended=$te groups=$g"; BBSI_TWO_ENDED=$te BBSI_GROUPS=$g timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k:(v['launches'],round(v['ms'],1)) for k,v in d['roofline']['kernels'].items()})"
done; done 2>&1 | tee gpurun_out/t2_bench.log
