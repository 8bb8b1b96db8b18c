set -u
mkdir -p gpurun_out
S=paper_2605_19910_b200/_lib/libbbsi_cuda_share.so
for i in 1 2 3 4 5 6; do
  timeout 300 python -m pytest tests/test_gpu_rgf.py -x -q -k "rgf_many" 2>&1 | tail -1 | sed "s/^/default $i: /" | tee -a gpurun_out/l_flaky.log
done
for i in 1 2 3 4 5 6; do
  BBSI_LIB=$S timeout 300 python -m pytest tests/test_gpu_rgf.py -x -q -k "rgf_many" 2>&1 | tail -1 | sed "s/^/share $i: /" | tee -a gpurun_out/l_flaky.log
done
BBSI_LIB=$S timeout 300 python - <<'PY' 2>&1 | tee -a gpurun_out/l_flaky.log
import sys
sys.path.insert(0, '.')
import numpy as np
from oracle import bbsi_oracle as O
from paper_2605_19910_b200 import bbsi as P
from tests._util import to_product
for rep in range(4):
    for li, lay in enumerate((O.make_layout(14, 9, 1), O.make_layout(16, 6, 2), O.BlockLayout(7, [3, 5, 2, 5, 4, 1, 5], 1))):
        ms = [to_product(O.random_spd_like(lay, 1300 + k, 2.0)) for k in range(4)]
        many = P.rgf_many(ms)
        single = P.rgf_ndiag if lay.bandwidth > 1 else P.rgf_tridiag
        for mi, (m, (g, c)) in enumerate(zip(ms, many)):
            g1, c1 = single(m)
            if not np.array_equal(g.data, g1.data):
                d = np.abs(g.data - g1.data)
                print(f"share rep {rep} layout {li} matrix {mi}: differ, max abs {d.max():.3e}, n differing {int((d > 0).sum())}, nan {int(np.isnan(g.data).sum())} {int(np.isnan(g1.data).sum())}")
PY
