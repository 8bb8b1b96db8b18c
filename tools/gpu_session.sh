#!/bin/bash
set -u
O=gpurun_out
echo "== pytest -m gpu"; timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
echo "== bench (full line)"; timeout 900 python bench.py > $O/bench_full3.json 2> $O/bench_full3.err; tail -1 $O/bench_full3.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['e2e'], d['cpu_baseline']['value'] if d['cpu_baseline'] else None)"
