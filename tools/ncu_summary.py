#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and/or a
--set full report into a markdown table (per-kernel share, occupancy, DRAM, tensor)."""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                agg[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | mean us | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / tot:.3f} |")
    return "\n".join(out)


WANT = {
    "Duration": "dur",
    "Achieved Occupancy": "occ%",
    "Registers Per Thread": "regs",
    "DRAM Throughput": "dram%",
    "Compute (SM) Throughput": "sm%",
    "Executed Ipc Active": "ipc",
    "Grid Size": "grid",
    "L2 Hit Rate": "l2hit%",
}


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = rows[0]
    per = collections.OrderedDict()
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"].split("(")[0])
        if d.get("Metric Name") in WANT:
            per.setdefault(key, {})[WANT[d["Metric Name"]]] = d["Metric Value"] + (
                " " + d["Metric Unit"] if d["Metric Name"] == "Duration" else "")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    h2 = rr[0]
    cols = {n: i for i, n in enumerate(h2)}
    extra = {}
    for r in rr[2:]:
        key = (r[cols["ID"]], r[cols["Kernel Name"]].split("(")[0])
        e = {}
        for name in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
                     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"):
            if name in cols:
                e[name] = r[cols[name]]
        extra[key] = e
    out = ["| id | kernel | " + " | ".join(WANT.values()) + " | dram rd (MB) | dram wr (MB) | dmma inst % of peak |",
           "|" + "---|" * (len(WANT) + 5)]
    for key, d in per.items():
        e = extra.get(key, {})
        dm = e.get("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "")
        out.append(f"| {key[0]} | `{key[1]}` | " + " | ".join(d.get(v, "") for v in WANT.values())
                   + f" | {mb(e.get('dram__bytes_read.sum'))} | {mb(e.get('dram__bytes_write.sum'))} | {dm} |")
    return "\n".join(out)


def mb(v):
    try:
        return f"{float(v.replace(',', '')) / 1e6:.3f}"
    except (AttributeError, ValueError):
        return ""


STAGE = {"k_synthesis": "legendre_synthesis", "k_ring": "ring_fft_products",
         "k_analysis": "legendre_analysis"}


def traffic(path):
    """{stage: dram read + write bytes of the largest captured launch of that kernel}."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    cols = {n: i for i, n in enumerate(rr[0])}
    out = {}
    for r in rr[2:]:
        name = r[cols["Kernel Name"]].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
        for prefix, stage in STAGE.items():
            if name.startswith(prefix):
                b = sum(float(r[cols[k]].replace(",", "")) for k in ("dram__bytes_read.sum",
                                                                      "dram__bytes_write.sum"))
                out[stage] = max(out.get(stage, 0.0), b)
    return out


if __name__ == "__main__":
    if sys.argv[1] == "--traffic":  # --traffic REPORT OUT.json
        import json

        with open(sys.argv[3], "w") as f:
            json.dump(traffic(sys.argv[2]), f, indent=1)
        sys.exit(0)
    for p in sys.argv[1:]:
        print(f"### {p}\n")
        print(launches(p) if p.endswith(".csv") else full(p))
        print()
