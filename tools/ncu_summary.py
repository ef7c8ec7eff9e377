"""Summarise ncu outputs into small text files for profiles/ (run here, no GPU).

    python tools/ncu_summary.py launches gpurun_out/launches_X.csv > profiles/..._launches.txt
    python tools/ncu_summary.py full gpurun_out/attn_X.ncu-rep > profiles/..._attn_full.txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.per_cycle_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sector_hit_rate.pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    # skip ncu preamble lines until the header
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            rows = rows[i:]
            break
    hdr = rows[0]
    ki = hdr.index("Kernel Name")
    vi = hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1.0)
        tot[name] += v * scale
        cnt[name] += 1
    allms = sum(tot.values())
    print(f"# ncu launch list {path}: {sum(cnt.values())} launches, {allms:.3f} ms total (serialised, cold)")
    print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'avg ms':>10s} {'share':>7s}")
    for name in sorted(tot, key=lambda k: -tot[k]):
        print(f"{name[:60]:60s} {cnt[name]:8d} {tot[name]:10.3f} {tot[name]/cnt[name]:10.4f} "
              f"{100*tot[name]/allms:6.2f}%")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary of {path}")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(f"\n## {d.get('Kernel Name', '?')[:120]}")
        for k in KEYS:
            if k in d:
                print(f"{k:70s} {d[k]:>20s} {units[hdr.index(k)]}")
        stalls = sorted(((k, float(d[k] or 0)) for k in hdr
                         if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")),
                        key=lambda x: -x[1])
        tot = sum(v for _, v in stalls) or 1.0
        print("top stall reasons (pc sampling):")
        for k, v in stalls[:8]:
            print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {100*v/tot:6.2f}%")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
