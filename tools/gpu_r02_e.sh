set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/e_kernels.log 2>&1; echo "kernel tests rc=$?"; tail -4 gpurun_out/e_kernels.log
for lib in libbbsi_cuda_dbg.so libbbsi_cuda_dbg2.so; do
  echo "== $lib" | tee -a gpurun_out/e_marks.log
  for cfg in "256 128" "256 2" "512 16" "768 2"; do
    set -- $cfg
    BBSI_LIB=paper_2605_19910_b200/_lib/$lib timeout 300 python tools/dbg_zinv_rows.py --block $1 --batch $2 2>&1 | tail -1 | tee -a gpurun_out/e_marks.log
  done
done
BBSI_LIB=paper_2605_19910_b200/_lib/libbbsi_cuda_dbg2.so timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k zinv 2>&1 | tail -2
