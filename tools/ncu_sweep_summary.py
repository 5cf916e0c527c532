"""Summarise tools/ncu_sweep.sh output: one row per (dtype, nrhs)."""
import csv
import re
import sys

print(f"{'dtype':5s} {'b':>3s} {'us':>8s} {'DRAM rd MB':>10s} {'DRAM wr MB':>10s} {'alg MB':>8s} {'traffic/alg':>11s} "
      f"{'L2 hit%':>7s} {'L2 rd hit%':>10s} {'TMA MB':>8s} {'LDG MB':>8s}  kernel")
n = 32 * 16 ** 3
for path in sys.argv[1:]:
    m = re.search(r"ncu_sweep_(c\d+)_b(\d+)\.csv", path)
    dt, b = m.group(1), int(m.group(2))
    w = 16 if dt == "c128" else 8
    d, kern = {}, ""
    for r in csv.DictReader(open(path)):
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1,
              "nsecond": 1e-3, "msecond": 1e3}.get(unit, 1)
        d[r["Metric Name"]] = v
        kern = r["Kernel Name"]
    alg = (24 * b + 36) * w * n
    rd, wr = d.get("dram__bytes_read.sum", 0), d.get("dram__bytes_write.sum", 0)
    print(f"{dt:5s} {b:3d} {d.get('gpu__time_duration.sum', 0):8.1f} {rd / 1e6:10.1f} {wr / 1e6:10.1f} {alg / 1e6:8.1f} "
          f"{(rd + wr) / alg:11.3f} {d.get('lts__t_sector_hit_rate.pct', 0):7.1f} "
          f"{d.get('lts__t_sector_op_read_hit_rate.pct', 0):10.1f} "
          f"{d.get('l1tex__m_xbar2l1tex_read_bytes.sum', 0) / 1e6:8.1f} "
          f"{d.get('l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum', 0) / 1e6:8.1f}  {kern[:60]}")
