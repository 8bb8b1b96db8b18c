# Round-2 call M: the SM-sharing panel as the default build (and the rgf_many H2D ordering fix):
# GPU suite, bit-identity against the exclusive build, the config-2 / 3 / 4 bench lines, ncu of the panel.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r02_gpu_tests.log
for lib in "" paper_2605_19910_b200/_lib/libbbsi_cuda_excl.so; do
  BBSI_LIB=$lib python - <<'PY' | tee -a gpurun_out/m_bits.log
import ctypes as C, hashlib, os, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2605_19910_b200._native import lib
for n in (128, 256, 512, 768):
    rng = np.random.default_rng(n)
    a = rng.uniform(-1, 1, (3, n, n)) + 1j * rng.uniform(-1, 1, (3, n, n))
    d = torch.from_numpy(a).cuda()
    st = np.zeros(3, dtype=np.int32)
    assert lib().bbsi_cuda_zinv_dev(n, n, 3, C.c_void_p(d.data_ptr()), n, n * n, st.ctypes.data_as(C.c_void_p), C.c_void_p(0)) == 0
    torch.cuda.synchronize()
    print(os.environ.get("BBSI_LIB") or "default", n, hashlib.sha1(d.cpu().numpy().tobytes()).hexdigest())
PY
done
for i in 1 2 3; do
  timeout 300 python - <<'PY' 2>&1 | tail -3 | tee -a gpurun_out/m_many.log
import sys
sys.path.insert(0, '.')
import numpy as np
from oracle import bbsi_oracle as O
from paper_2605_19910_b200 import bbsi as P
from tests._util import to_product
bad = 0
for rep in range(4):
    for li, lay in enumerate((O.make_layout(14, 9, 1), O.make_layout(16, 6, 2), O.BlockLayout(7, [3, 5, 2, 5, 4, 1, 5], 1))):
        ms = [to_product(O.random_spd_like(lay, 1300 + k, 2.0)) for k in range(4)]
        many = P.rgf_many(ms)
        single = P.rgf_ndiag if lay.bandwidth > 1 else P.rgf_tridiag
        for mi, (m, (g, c)) in enumerate(zip(ms, many)):
            g1, c1 = single(m)
            bad += not np.array_equal(g.data, g1.data)
print("rgf_many vs single calls, 4 reps x 3 layouts x 4 matrices: mismatches", bad)
PY
done
python bench.py > gpurun_out/r02_bench_cfg2.json 2> gpurun_out/r02_bench_cfg2.err; echo "cfg2 rc=$?"
python bench.py --config 3 > gpurun_out/r02_bench_cfg3.json 2> gpurun_out/r02_bench_cfg3.err; echo "cfg3 rc=$?"
python bench.py --config 4 > gpurun_out/r02_bench_cfg4.json 2> gpurun_out/r02_bench_cfg4.err; echo "cfg4 rc=$?"
BBSI_LIB=paper_2605_19910_b200/_lib/libbbsi_cuda_excl.so python bench.py --no-e2e --no-cpu-baseline --no-traffic > gpurun_out/r02_cfg2_exclusive.json 2> gpurun_out/r02_cfg2_exclusive.err; echo "excl rc=$?"
export BBSI_GRAPHS=0 BBSI_GROUPS=1
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:gj_rows_kernel" -s 24 -c 1 -o gpurun_out/r02_full_gjrows \
    python tools/prof_step.py --config 2 --layers 64 --energies 64 --reps 1 > gpurun_out/r02_full_gjrows.log 2>&1; echo "ncu rc=$?"
unset BBSI_GRAPHS BBSI_GROUPS
python bench.py --config 5 --steps 1 --warmup 3 > gpurun_out/r02_bench_cfg5.json 2> gpurun_out/r02_bench_cfg5.err; echo "cfg5 rc=$?"
