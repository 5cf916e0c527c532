"""Summarise an ncu report into profiles/: key metrics per kernel launch.

python tools/ncu_summary.py gpurun_out/x.ncu-rep profiles/name.json [--alg-bytes N]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
    "launch__shared_mem_per_block_dynamic",
]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    alg = None
    if "--alg-bytes" in sys.argv:
        alg = float(sys.argv[sys.argv.index("--alg-bytes") + 1])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        e = {"kernel": d.get("Kernel Name"), "id": d.get("ID")}
        for k in KEYS:
            if k in d:
                try:
                    v = float(d[k].replace(",", ""))
                except ValueError:
                    v = d[k]
                e[k] = v
                e[k + ".unit"] = u.get(k)
        # normalise bytes to bytes
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            unit = e.get(k + ".unit", "")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            if isinstance(e.get(k), float):
                e[k + ".bytes"] = e[k] * scale
        if "dram__bytes_read.sum.bytes" in e:
            e["dram_traffic_bytes"] = e["dram__bytes_read.sum.bytes"] + e["dram__bytes_write.sum.bytes"]
            if alg:
                e["algorithmic_bytes"] = alg
                e["traffic_over_algorithmic"] = e["dram_traffic_bytes"] / alg
        res.append(e)
    json.dump({"report": rep, "launches": res}, open(out, "w"), indent=1)
    for e in res:
        print(e["kernel"][:90], e.get("gpu__time_duration.sum"), e.get("dram_traffic_bytes"))


if __name__ == "__main__":
    main()
