"""Per-position timing of the Gauss-Jordan launches in an ncu launch list: pair-panel and
GJ-GEMM mean duration by step index inside one inversion (step 0 reads the input block)."""
import collections
import csv
import sys


def main(path):
    hdr, data = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    pos, gpos = collections.defaultdict(list), collections.defaultdict(list)
    k = 0
    for d in data:
        name = d["Kernel Name"].split("(")[0].split("::")[-1]
        t = float(d["Metric Value"]) / 1e3
        if name.startswith("gj_pair"):
            pos[k].append(t)
        elif name.startswith("zgemm_grouped_kernel<1"):
            gpos[k].append(t)
            k += 1
        else:
            k = 0
    for k in sorted(pos):
        g = gpos.get(k, [0.0])
        print(f"step {k}: pair n={len(pos[k])} mean={sum(pos[k]) / len(pos[k]):.1f} us   "
              f"gj_gemm mean={sum(g) / len(g):.1f} us")


if __name__ == "__main__":
    main(sys.argv[1])
