#!/bin/bash
set -u
O=gpurun_out
echo "== pytest -m gpu"; timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
B="python bench.py --no-e2e --no-cpu-baseline --steps 3 --warmup 3"
echo "== bench default";        timeout 600 $B 2>&1 | tail -1 | cut -c1-200
P="python tools/prof_step.py --config 2 --layers 8 --energies 64"
N="ncu --metrics gpu__time_duration.sum --clock-control none --csv"
echo "== launches groups 1"
BBSI_GROUPS=1 timeout 300 $P > /dev/null 2>&1 && BBSI_GROUPS=1 timeout 600 $N --log-file $O/ll.csv $P > /dev/null 2>&1
python tools/launches.py $O/ll.csv > $O/ll.txt; head -6 $O/ll.txt
echo "== accuracy";             timeout 900 python tools/accuracy_probe.py --config 3 --energies 17 2>&1 | tail -1
