set -u
O=gpurun_out
P="python tools/prof_step.py --config 2 --layers 8 --energies 64"
export BBSI_GROUPS=1
timeout 300 $P > /dev/null 2>&1 || echo "prof_step failed"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gj_panel_rows --launch-skip 20 -c 1 -o $O/panel_rows -f $P > $O/ncu_panel.log 2>&1; tail -2 $O/ncu_panel.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:zgemm_grouped_kernel --launch-skip 40 -c 1 -o $O/gj_gemm -f $P > $O/ncu_gjgemm.log 2>&1; tail -2 $O/ncu_gjgemm.log
