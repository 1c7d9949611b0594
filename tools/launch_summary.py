"""Per-kernel share of one solve from an ncu launch list (gpu__time_duration.sum).

usage: python tools/launch_summary.py launches.csv [--solves 2] > profiles/rNN_ncu_launches_<cfg>.txt
The capture runs tools/profile_solve.py --solves S; only the LAST solve's
launches are summarised (the first one includes uploads and warm-up).
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    solves = int(sys.argv[sys.argv.index("--solves") + 1]) if "--solves" in sys.argv else 2
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    seq = []
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(r[ui], 1.0)
        seq.append((r[ki], v))
    # split solves at the pair-filter launch (first kernel of each solve)
    marks = [i for i, (k, _) in enumerate(seq) if "k_enumerate_pairs" in k]
    last = seq[marks[-1]:] if len(marks) >= solves else seq
    tot = sum(v for _, v in last)
    agg = collections.OrderedDict()
    for k, v in last:
        name = k.split("(")[0][:62]
        a = agg.setdefault(name, [0.0, 0])
        a[0] += v
        a[1] += 1
    print(f"ncu --metrics gpu__time_duration.sum --clock-control none, tools/profile_solve.py, {solves} solves")
    print(f"last solve: {len(last)} launches, {tot:.3f} ms of kernel time (ncu serialised, cold caches)")
    for name, (v, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{name:62s} {v:8.3f} ms  {100 * v / tot:5.1f}%  n={n}")


if __name__ == "__main__":
    main()
