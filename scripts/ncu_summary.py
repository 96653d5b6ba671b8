"""Summarise ncu reports (gpurun_out/*.ncu-rep) into a markdown table:
duration, DRAM bytes and throughput, L1TEX/L2 throughput, occupancy."""
import csv
import io
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "dur_us",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "dram__cycles_active.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_hz",
    "l1tex__t_sector_hit_rate.pct": "l1_hit",
    "lts__t_sector_hit_rate.pct": "l2_hit",
}


def raw(path):
    """One dict per profiled kernel of the report."""
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, vals):
            if h in WANT:
                scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1.0, "KB": 1e3, "MB": 1e6,
                         "GB": 1e9, "hz": 1.0, "Mhz": 1e6, "Ghz": 1e9, "Hz": 1.0, "MHz": 1e6, "GHz": 1e9}.get(u, 1.0)
                try:
                    d[WANT[h]] = float(v.replace(",", "")) * scale
                except ValueError:
                    pass
            if h == "Kernel Name":
                d["kernel"] = v
        res.append(d)
    return res


print("| report | # | kernel | time (us) | DRAM read+write (MB) | DRAM % peak | L1TEX % | L2 % | L1 hit % | L2 hit % | warps active % | SM clock (MHz) |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
for p in sys.argv[1:]:
    name = p.rsplit("/", 1)[-1].replace(".ncu-rep", "")
    for i, d in enumerate(raw(p)):
        tot = (d.get("dram_rd", 0) + d.get("dram_wr", 0)) / 1e6
        print(f"| {name} | {i} | `{d.get('kernel', '?')[:44]}` | {d.get('dur_us', 0):.1f} | {tot:.1f} | "
              f"{d.get('dram_pct', 0):.1f} | {d.get('l1tex_pct', 0):.1f} | {d.get('l2_pct', 0):.1f} | "
              f"{d.get('l1_hit', 0):.1f} | {d.get('l2_hit', 0):.1f} | {d.get('occ_pct', 0):.1f} | "
              f"{d.get('sm_hz', 0) / 1e6:.0f} |")
