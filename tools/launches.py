"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import collections
import csv
import sys


def load(path):
    hdr, data = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


def main(path, show=0):
    data = load(path)
    agg = collections.defaultdict(list)
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
        key = f"{name} grid={d.get('Grid Size', '')}"
        agg[key].append(float(d["Metric Value"]) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    print(f"{len(data)} launches, {tot:.1f} us total (cold-cache, serialised)")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {sum(v):10.1f} us {100 * sum(v) / tot:5.1f}%  n={len(v):5d} mean={sum(v) / len(v):8.2f} us  {k}")
    for d in data[:show]:
        print(d["Kernel Name"][:50], float(d["Metric Value"]) / 1e3, d.get("Grid Size"))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
