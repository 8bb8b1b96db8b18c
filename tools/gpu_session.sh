#!/bin/bash
set -u
echo "== gpu tests"; timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
B="python bench.py --no-e2e --no-cpu-baseline --steps 3 --warmup 3"
echo "== bench"; timeout 600 $B 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step']); print(json.dumps(d['roofline']['kernels']))"
