#!/usr/bin/env python
"""Summarise ncu output for profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py launches <launches.csv> [--step-kernels N]
    python tools/ncu_summary.py report <prof.ncu-rep>

`launches` prints the per-launch device times of one learner step (the last complete
step in the capture) and each kernel's share; `report` prints, per profiled kernel,
duration, DRAM bytes, tensor-pipe and memory utilisation, occupancy and registers.
"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict


def short(name):
    name = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    if "gemm_tf32x3_kernel" in name:
        return "gemm_tf32x3" + name[name.index("<"):name.index(">") + 1]
    return name.split("(")[0].replace("void ", "").replace("tlg::", "")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
    ks = [(int(r[ii]), short(r[ki]), float(r[vi].replace(",", ""))) for r in rows[hi + 1:]
          if len(r) > vi]
    # one step = from an optimizer launch (exclusive) to the next optimizer launch (inclusive)
    opt = [i for i, k in enumerate(ks) if "optimizer" in k[1]]
    lo, hi_ = (opt[-2] + 1, opt[-1] + 1) if len(opt) >= 2 else (0, len(ks))
    step = ks[lo:hi_]
    tot = sum(k[2] for k in step)
    print(f"| # | kernel | us | share |\n|---|---|---|---|")
    for i, (_, n, t) in enumerate(step):
        print(f"| {i} | `{n}` | {t / 1e3:.1f} | {100 * t / tot:.1f}% |")
    print(f"| | **step total (serialised, cold-cache)** | **{tot / 1e3:.1f}** | |")


WANT = OrderedDict([
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm %"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum.per_second", "L2->SM"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
])


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    idx = {k: h.index(k) for k in WANT if k in h}
    print("| kernel | " + " | ".join(WANT[k] for k in idx) + " |")
    print("|---|" + "---|" * len(idx))
    for r in rows[2:]:
        cells = []
        for k, i in idx.items():
            u = units[i]
            cells.append(f"{r[i]} {u}".strip())
        print(f"| `{short(r[h.index('Kernel Name')])}` | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[2])
