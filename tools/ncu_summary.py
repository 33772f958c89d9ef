"""Per-kernel summary of an ncu --set full report: duration, DRAM bytes, throughput, occupancy, top stalls."""
import csv
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[2:]


def f(d, k):
    try:
        return float(d.get(k, "nan").replace(",", ""))
    except ValueError:
        return float("nan")


def main(rep):
    h, rows = raw(rep)
    for row in rows:
        d = dict(zip(h, row))
        name = d.get("Kernel Name", "")[:48]
        t = f(d, "gpu__time_duration.sum")
        rd, wr = f(d, "dram__bytes_read.sum"), f(d, "dram__bytes_write.sum")
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v.replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        pipes = sorted((k, v) for k, v in d.items()
                       if k.startswith("sm__pipe_") and k.endswith("_cycles_active.avg.pct_of_peak_sustained_active")
                       and v not in ("0", "0.000000"))
        print(f"{name:48s} t={t} dram_rd={rd} dram_wr={wr} "
              f"dram%={f(d, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} "
              f"l2hit={f(d, 'lts__t_sector_hit_rate.pct'):.1f} occ={f(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} "
              f"regs={d.get('launch__registers_per_thread')} stalls={[(round(a, 2), b) for a, b in stalls[:4]]}")
        if pipes:
            print("    pipes: " + ", ".join(f"{k[len('sm__pipe_'):-len('_cycles_active.avg.pct_of_peak_sustained_active')]}={v}%" for k, v in pipes))


if __name__ == "__main__":
    main(sys.argv[1])
