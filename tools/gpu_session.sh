#!/bin/bash
# One GPU session: parity suite, bench variants, accuracy probe, panel timing breakdown.
# Usage (on the box): bash tools/gpu_session.sh > gpurun_out/session.log 2>&1
set -u
O=gpurun_out
mkdir -p $O
echo "== pytest -m gpu"; timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
B="python bench.py --no-e2e --no-cpu-baseline --steps 3 --warmup 3"
echo "== bench default";       timeout 600 $B 2>&1 | tail -1
echo "== bench graphs off";    BBSI_GRAPHS=0 timeout 600 $B 2>&1 | tail -1
echo "== bench groups 2";      BBSI_GROUPS=2 timeout 600 $B 2>&1 | tail -1
echo "== bench groups 2 nopri"; BBSI_GROUPS=2 BBSI_PANEL_PRIORITY=0 timeout 600 $B 2>&1 | tail -1
echo "== bench nb32";          BBSI_GJ_NB=32 timeout 600 $B 2>&1 | tail -1
echo "== accuracy nb16";       timeout 900 python tools/accuracy_probe.py --config 3 --energies 17 2>&1 | tail -6
echo "== accuracy nb32";       BBSI_GJ_NB=32 timeout 900 python tools/accuracy_probe.py --config 3 --energies 17 2>&1 | tail -6
echo "== panel breakdown";     BBSI_LIB=$PWD/paper_2605_19910_b200/_lib/libbbsi_cuda_dbg.so timeout 300 python tools/dbg_zinv.py 2>&1 | tail -8
