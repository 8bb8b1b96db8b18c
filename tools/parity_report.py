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
    solves = [r for r in rows if "max" in r]
    for r in solves:  # config 5: the input-noise floors come from the CPU floor run
        if r["config"] == 5 and r.get("floor") is None and r["energy_index"] in floors5:
            r["floor"] = floors5[r["energy_index"]]["floor"]
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
                  else (f"{fl:.2e}" if fl is not None else "—"))
            print(f"| {r['energy_index']} | {r['E']:+.4f} | {r['max']:.2e} | {r['median']:.2e} | {fs} | "
                  f"{r['residual_gpu']:.1e} / {r['residual_ref']:.1e} | {r.get('verdict', '?')} |")
        print()
    if floors5:
        print("### config 5 input-noise floors (CPU, streaming reference on A vs perturbed A)\n")
        print("| energy | E | floor | median |")
        print("|---|---|---|---|")
        for e, r in sorted(floors5.items()):
            print(f"| {e} | {r['E']:+.4f} | {r['floor']:.2e} | {r['floor_median']:.2e} |")


if __name__ == "__main__":
    main()
