#!/bin/bash
set -u
for p in 0 1; do echo "== group priority $p"; BBSI_GROUP_PRIORITY=$p timeout 900 python bench.py --no-cpu-baseline --steps 2 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'])"; done
