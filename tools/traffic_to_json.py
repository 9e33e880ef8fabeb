"""Pair tools/traffic_capture.py's launch labels with an ncu CSV of the same
run and write profiles/ncu_traffic_r02.json: per config, "kernel:nbN" ->
DRAM bytes (read + write) of that launch.

python tools/traffic_to_json.py capture.log ncu.csv [out.json]"""
import csv
import io
import json
import sys
from collections import OrderedDict


def rows(path):
    text = open(path).read()
    start = text.find('"ID"')
    data = list(csv.DictReader(io.StringIO(text[start:])))
    launches = OrderedDict()
    for r in data:
        key = (r["ID"], r["Kernel Name"])
        d = launches.setdefault(key, {})
        val = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(unit, 1)
        d[r["Metric Name"]] = val * scale
        d["kernel"] = r["Kernel Name"]
    return list(launches.values())


def main(log, csv_path, out="profiles/ncu_traffic_r02.json"):
    labels = []
    for line in open(log):
        if line.startswith("SKIP "):
            labels += [None] * int(line.split()[1])
        elif line.startswith("LAUNCH "):
            labels.append(line.split()[1])
    launches = rows(csv_path)
    if len(launches) != len(labels):
        raise SystemExit(f"{len(launches)} profiled launches vs {len(labels)} labels")
    res = {"source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum(,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum) of tools/traffic_capture.py "
                     f"(live states, one launch per label; cold L2 per ncu replay); {csv_path}"}
    for lab, d in zip(labels, launches):
        if lab is None:
            continue
        cfg, kern, nb = lab.split(":")
        # a label repeated by consecutive launches (the H-free stages' two kernels) sums them
        r = res.setdefault(cfg, {})
        key = f"{kern}:{nb}"
        r[key] = r.get(key, 0.0) + d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        wf = d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
        if wf is not None:  # shared-memory wavefronts (128 B each): the on-chip traffic
            r[key + ":smem_wavefronts"] = r.get(key + ":smem_wavefronts", 0.0) + wf
        r[key + ":kernel"] = (r[key + ":kernel"] + " + " if key + ":kernel" in r else "") + d["kernel"][:80]
        r[key + ":ncu_us"] = r.get(key + ":ncu_us", 0.0) + d.get("gpu__time_duration.sum", 0) / 1e3
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
