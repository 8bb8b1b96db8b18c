#!/bin/bash
# Round-1 evidence: parity suite, full bench line, bench launch list, top-kernel profile.
set -u
O=gpurun_out
echo "== pytest -m gpu"; timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
echo "== bench (full line)"; timeout 900 python bench.py > $O/bench_full.json 2> $O/bench_full.err; tail -1 $O/bench_full.json | cut -c1-300
C="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
echo "== bench launch list"
timeout 900 $C > $O/plain_bench.log 2>&1 && timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 20000 -c 600 --csv --log-file $O/launches_bench.csv $C > $O/ncu_bench.log 2>&1
python tools/launches.py $O/launches_bench.csv > $O/launches_bench.txt; head -8 $O/launches_bench.txt
P="python tools/prof_step.py --config 2 --layers 8 --energies 64"
echo "== top kernel full profile"
BBSI_GROUPS=1 timeout 300 $P > $O/plain_prof.log 2>&1 && BBSI_GROUPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:zgemm_grouped_kernel -s 17 -c 1 -o $O/r01_zgemm_main -f $P > $O/ncu_zgemm.log 2>&1; tail -1 $O/ncu_zgemm.log
BBSI_GROUPS=1 timeout 300 $P > $O/plain_prof2.log 2>&1 && BBSI_GROUPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:gj_panel_rows -s 20 -c 1 -o $O/r01_panel -f $P > $O/ncu_panel.log 2>&1; tail -1 $O/ncu_panel.log
