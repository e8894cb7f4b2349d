"""Summaries of ncu captures for profiles/ (dev tool).

python tools/summarize_ncu.py launches <launches.csv>          # per-kernel share of device time
python tools/summarize_ncu.py full <report.ncu-rep> [label]    # key counters + stall/line attribution
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        name = r[4].split("(")[0].split("<")[0].strip()
        if "traverse_kernel" in r[4]:
            name = r[4].split("(")[0].strip()
        if r[12] == "gpu__time_duration.sum":
            tot[name] += float(r[14]) / 1e3
            cnt[name] += 1
    allt = sum(tot.values())
    print(f"# ncu launch list ({path}); gpu__time_duration.sum, --clock-control none")
    print(f"# cold-cache, serialised launches: compare SHARES, not absolute times")
    print(f"{'kernel':70s} {'launches':>8s} {'total_us':>12s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k[:70]:70s} {cnt[k]:8d} {v:12.1f} {100 * v / allt:6.1f}%")


def full(rep, label=""):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "launch__occupancy_limit_registers", "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum",
            "l1tex__m_l1tex2xbar_write_sectors_mem_global_op_atom.sum",
            "l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum",
            "lts__t_sectors.sum", "lts__t_requests.sum",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum"]
    print(f"# ncu --set full --clock-control none: {label or rep}")
    for r in rows[2:]:
        for w in want:
            if w in hdr:
                i = hdr.index(w)
                print(f"{w:60s} {r[i]} {units[i]}")
    try:
        i = hdr.index("gpu__time_duration.sum")
        t_ms = float(rows[2][i]) if units[i] == "ms" else float(rows[2][i]) / 1e3
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
        rd = float(rows[2][hdr.index("dram__bytes_read.sum")]) * \
            scale[units[hdr.index("dram__bytes_read.sum")]]
        wr = float(rows[2][hdr.index("dram__bytes_write.sum")]) * \
            scale[units[hdr.index("dram__bytes_write.sum")]]
        print(f"{'derived: dram read+write bytes':60s} {rd + wr:.4e}")
        print(f"{'derived: achieved DRAM GB/s':60s} {(rd + wr) / (t_ms * 1e-3) / 1e9:.1f}")
        for nm, lab in (("l1tex__m_l1tex2xbar_write_sectors_mem_global_op_atom.sum", "atomic"),
                        ("l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum", "reduction")):
            if nm in hdr:
                x = float(rows[2][hdr.index(nm)].replace(",", ""))
                print(f"{'derived: global ' + lab + ' sectors to L2 per second (G)':60s} "
                      f"{x / (t_ms * 1e-3) / 1e9:.2f}")
        if "lts__t_sectors.sum" in hdr:
            x = float(rows[2][hdr.index("lts__t_sectors.sum")].replace(",", ""))
            print(f"{'derived: L2 sectors per second (G)':60s} {x / (t_ms * 1e-3) / 1e9:.1f}")
    except (ValueError, KeyError, IndexError):
        pass
    print()
    print("# stall attribution by CUDA source line (tools/ncu_lines.py)")
    print(subprocess.run([sys.executable, "tools/ncu_lines.py", rep, "25"], capture_output=True,
                         text=True).stdout)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
