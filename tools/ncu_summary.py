"""Summarise ncu captures into profiles/: key metrics of a --set full report (.ncu-rep) or the
per-launch time list of a --metrics gpu__time_duration.sum CSV.

  python tools/ncu_summary.py full gpurun_out/prof.ncu-rep profiles/r1_dense_pair.json
  python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r1_launches.json
"""

import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "smsp__inst_executed.sum", "launch__cluster_dim_x",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sectors_srcunit_tex.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "Tbyte": 1e12}


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        rec = {"kernel": vals[hdr.index("Kernel Name")]}
        for h, u, v in zip(hdr, units, vals):
            if h in KEYS:
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                rec[h] = {"value": x, "unit": u}
        rb = rec.get("dram__bytes_read.sum")
        wb = rec.get("dram__bytes_write.sum")
        if rb and wb:
            rec["dram_bytes_per_launch"] = rb["value"] * SCALE.get(rb["unit"], 1) + \
                wb["value"] * SCALE.get(wb["unit"], 1)
        kernels.append(rec)
    json.dump({"source": rep, "kernels": kernels}, open(out, "w"), indent=1)
    for k in kernels:
        print(k["kernel"][:80], {h: k[h]["value"] for h in k if isinstance(k[h], dict)})


def launches(path, out):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    items = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        items.append({"id": int(r["ID"]), "kernel": r["Kernel Name"][:120],
                      "time": float(r["Metric Value"].replace(",", "")),
                      "unit": r["Metric Unit"]})
    total = sum(i["time"] for i in items) or 1.0
    by = {}
    for i in items:
        name = i["kernel"].split("(")[0]
        by[name] = by.get(name, 0.0) + i["time"]
    share = {k: v / total for k, v in sorted(by.items(), key=lambda kv: -kv[1])}
    json.dump({"source": path, "launches": items, "share_of_device_time": share}, open(out, "w"),
              indent=1)
    for k, v in share.items():
        print(f"{v * 100:6.2f}%  {k}")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
