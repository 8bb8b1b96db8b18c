#!/bin/bash
set -u
O=gpurun_out
echo "== kernels"; timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu 2>&1 | tail -3
echo "== pytest -m gpu"; timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
B="python bench.py --no-e2e --no-cpu-baseline --steps 3 --warmup 3"
for v in 1 3; do echo "== bench panel $v"; BBSI_PANEL=$v timeout 600 $B 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step']); print(json.dumps(d['roofline']['kernels']))"; done
echo "== accuracy"; timeout 900 python tools/accuracy_probe.py --config 3 --energies 17 2>&1 | tail -1
