"""Summarise full-size parity records (tools/parity_full.py JSON lines) as markdown.

  python tools/parity_report.py profiles/r02_parity_*.jsonl > profiles/r02_parity_tables.md
"""
import collections
import json
import sys


def main():
    rows = []
    for path in sys.argv[1:]:
        for line in open(path):
            line = line.strip()
            if line.startswith("{"):
                r = json.loads(line)
                r["_file"] = path
                rows.append(r)
    floors5 = {r["energy_index"]: r for r in rows if r.get("kind") == "floor"}
    floors5b = {r["energy_index"]: r for r in rows if r.get("kind") == "floor_blas"}
    solves = [r for r in rows if "max" in r]
    for r in solves:  # config 5: the floors come from the CPU floor runs (input noise; BLAS kernel order)
        e = r["energy_index"]
        if r["config"] == 5 and (e in floors5 or e in floors5b):
            fi = floors5[e]["floor"] if e in floors5 else None
            fb = floors5b[e]["floor"] if e in floors5b else None
            r["floor_input"], r["floor_blas"] = fi, fb
            r["floor"] = max(x for x in (fi, fb) if x is not None)
            r["verdict"] = "<= 1e-10" if r["max"] <= 1e-10 else ("<= floor" if r["max"] <= r["floor"] else "ABOVE")
    by = collections.defaultdict(list)
    for r in solves:
        by[(r["config"], r["solver"])].append(r)
    print("| config | solver | energies | worst max error | verdicts | worst max / floor | GPU residual (max) | "
          "reference residual (max) |")
    print("|---|---|---|---|---|---|---|---|")
    for (k, solver), rs in sorted(by.items()):
        v = collections.Counter(r.get("verdict", "?") for r in rs)
        ratio = max((r["max"] / r["floor"]) for r in rs if r.get("floor")) if any(r.get("floor") for r in rs) else None
        print(f"| {k} | {solver} | {len(rs)} | {max(r['max'] for r in rs):.2e} | "
              + ", ".join(f"{n} {c}" for c, n in sorted(v.items()))
              + f" | {ratio:.2f} |" if ratio is not None else " | — |", end="")
        print(f" {max(r['residual_gpu'] for r in rs):.1e} | {max(r['residual_ref'] for r in rs):.1e} |")
    print()
    for (k, solver), rs in sorted(by.items()):
        print(f"### config {k}, {solver}\n")
        print("| energy | E | max | median | floor (input / BLAS) | residual GPU / ref | verdict |")
        print("|---|---|---|---|---|---|---|")
        for r in sorted(rs, key=lambda r: r["energy_index"]):
            fi, fb = r.get("floor_input"), r.get("floor_blas")
            fl = r.get("floor")
            fs = (f"{fl:.2e} ({fi:.2e} / {fb:.2e})" if fi is not None and fb is not None
                  else (f"{fl:.2e} ({fi:.2e} / —)" if fi is not None else (f"{fl:.2e}" if fl is not None else "—")))
            print(f"| {r['energy_index']} | {r['E']:+.4f} | {r['max']:.2e} | {r['median']:.2e} | {fs} | "
                  f"{r['residual_gpu']:.1e} / {r['residual_ref']:.1e} | {r.get('verdict', '?')} |")
        print()
    if floors5:
        print("### config 5 floors (CPU, streaming reference): input noise (A vs one-ulp-perturbed A) and BLAS "
              "kernel order (native AVX-512 kernels vs OPENBLAS_CORETYPE=Haswell, tools/cfg5_blas_floor.py)\n")
        print("| energy | E | input floor (max / median) | BLAS floor (max / median) |")
        print("|---|---|---|---|")
        for e, r in sorted(floors5.items()):
            fb = floors5b.get(e)
            fbs = f"{fb['floor']:.2e} / {fb['floor_median']:.2e}" if fb else "—"
            print(f"| {e} | {r['E']:+.4f} | {r['floor']:.2e} / {r['floor_median']:.2e} | {fbs} |")


if __name__ == "__main__":
    main()
