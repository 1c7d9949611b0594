"""Summarise an `ncu --set full` capture into a small JSON for profiles/.

usage: python tools/ncu_summary.py REPORT.ncu-rep OUT.json [--label TEXT]
Reads `ncu -i --page raw --csv` (metrics) and `--page source --print-source sass`
(stall reasons, instruction mix).  `traffic_bytes` = dram read + write of the
captured launch; bench.py quotes it as roofline.traffic.
"""
import collections
import csv
import io
import json
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
SCALE = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
         "Gbyte": 1e9}


def _csv(args):
    out = subprocess.run([NCU, "-i", *args], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def _stall_lines(rep, top=12):
    """Warp-stall samples per CUDA source line (needs -lineinfo), top lines."""
    rows = _csv([rep, "--page", "source", "--csv", "--print-source", "cuda,sass"])
    agg, fname, tot = collections.Counter(), "", 0
    text = {}
    for r in rows:
        if r and r[0] in ("File Path", "File Name"):
            fname = r[1].split("/")[-1]
            continue
        if len(r) < 6 or not r[0] or r[0] == "Line No":
            continue
        try:
            v = int(r[4])
        except ValueError:
            continue
        key = f"{fname}:{r[0]}"
        agg[key] += v
        text[key] = r[1].strip()[:80]
        tot += v
    tot = tot or 1
    return [{"line": k, "pct": round(100 * v / tot, 1), "source": text[k]} for k, v in agg.most_common(top)]


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    label = sys.argv[sys.argv.index("--label") + 1] if "--label" in sys.argv else ""
    raw = _csv([rep, "--page", "raw", "--csv"])
    hdr, units, vals = raw[0], raw[1], raw[2]
    res = {"report": rep.split("/")[-1], "label": label,
           "kernel": vals[hdr.index("Kernel Name")]}
    for k, name in KEYS.items():
        if k in hdr:
            i = hdr.index(k)
            v = float(vals[i].replace(",", ""))
            u = units[i]
            if name == "duration":
                res["duration_s"] = v * SCALE.get(u, 1.0)
            elif u in SCALE and name in ("dram_read", "dram_write", "l2_bytes"):
                res[name + "_bytes"] = v * SCALE[u]
            else:
                res[name] = v
    res["traffic_bytes"] = res.get("dram_read_bytes", 0) + res.get("dram_write_bytes", 0)
    if "duration_s" in res:
        res["dram_gbs"] = res["traffic_bytes"] / res["duration_s"] / 1e9
    rows = _csv([rep, "--page", "source", "--csv", "--print-source", "sass"])
    h = rows[1]
    ix = {x: i for i, x in enumerate(h)}
    stalls = collections.Counter()
    mix = collections.Counter()
    tot = 0.0
    for r in rows[2:]:
        try:
            n = float(r[ix["Instructions Executed"]])
        except (ValueError, IndexError):
            continue
        toks = r[ix["Source"]].split()
        if toks and toks[0].startswith("@"):
            toks = toks[1:]
        if toks:
            mix[toks[0].split(".")[0]] += n
        tot += n
        for k, i in ix.items():
            if k.startswith("stall_") and "Not Issued" not in k:
                try:
                    stalls[k[6:]] += float(r[i])
                except ValueError:
                    pass
    st = sum(stalls.values()) or 1.0
    res["stall_pct"] = {k: round(100 * v / st, 1) for k, v in stalls.most_common(8)}
    res["inst_mix_pct"] = {k: round(100 * v / tot, 1) for k, v in mix.most_common(10)}
    res["stall_lines_pct"] = _stall_lines(rep)
    with open(dst, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
