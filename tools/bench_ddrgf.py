"""DDRGF on one B200: BASELINE config 4 (l = 4096, b = 256, one energy) and a config 5
slice, timed against the batched sequential RGF on the same matrix.

  python tools/bench_ddrgf.py [--config 4] [--domains 2 4 8] [--reps 3]

Prints one JSON line per (solver, domains): ms per solve and selected inversions/s
(layers / s). The domains all run on this GPU (phase 1 / 3 batched over domains, phase 2
sequential over separators); across GPUs the same protocol shards domains
(paper_2605_19910_b200/distributed.py).
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=4)
    p.add_argument("--layers", type=int, default=0, help="override l (config 5: 512 keeps A + G + scratch in HBM)")
    p.add_argument("--domains", type=int, nargs="+", default=[2, 4, 8])
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--plans", nargs="*", default=[], help="DomainPlan s2_levels, e.g. 127 127,5 (A formed once)")
    a = p.parse_args()
    import torch

    from paper_2605_19910_b200 import dyson as D

    cfg = D.CONFIGS[a.config]
    if a.layers:
        cfg = D.scaled(cfg, num_layers=a.layers)
    l, b = cfg.num_layers, cfg.block_size
    H = torch.empty((l, 3, b, b), dtype=torch.complex128, device="cuda")
    D.fill_h_device(cfg, H)
    G = torch.empty((1, l, 3, b, b), dtype=torch.complex128, device="cuda")
    z = cfg.z()[:1]
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(a.reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.reps

    ms = timed(lambda: D.solve_device(cfg, H, G, z=z, stream=st))
    print(json.dumps({"config": cfg.name, "solver": "rgf (1 energy)", "layers": l, "block": b,
                      "ms": round(ms, 2), "inversions_per_s": round(l / (ms * 1e-3), 1)}), flush=True)
    G1 = G[0]
    if a.plans:
        import ctypes as C

        import numpy as np

        from paper_2605_19910_b200._native import lib

        A = H.neg()
        dg = A[:, 1].diagonal(dim1=-2, dim2=-1)
        sig = torch.from_numpy(cfg.sigma()).to(A.device)
        dg.copy_((complex(z[0]) + dg) - sig[:, None])
        for plan in a.plans:
            lv = np.array([int(x) for x in plan.split(",")], dtype=np.int32)
            fail = C.c_int(-1)

            def run():
                rc = lib().bbsi_cuda_ddrgf_plan_dev(l, b, lv.ctypes.data_as(C.c_void_p), len(lv),
                                                    C.c_void_p(A.data_ptr()), C.c_void_p(G1.data_ptr()),
                                                    C.byref(fail), C.c_void_p(st.cuda_stream))
                assert rc == 0, lib().bbsi_cuda_last_error()

            ms = timed(run)
            print(json.dumps({"config": cfg.name, "solver": f"ddrgf plan {plan} on 1 GPU", "layers": l, "block": b,
                              "ms": round(ms, 2), "inversions_per_s": round(l / (ms * 1e-3), 1)}), flush=True)
        return
    for P in a.domains:
        s2 = l // P - 1
        ms = timed(lambda: D.solve_ddrgf_device(cfg, H, G1, s2, stream=st))
        print(json.dumps({"config": cfg.name, "solver": f"ddrgf P={P} (s2={s2}) on 1 GPU", "layers": l, "block": b,
                          "ms": round(ms, 2), "inversions_per_s": round(l / (ms * 1e-3), 1)}), flush=True)


if __name__ == "__main__":
    main()
