"""Top SASS lines of one kernel in an ncu report (source page, csv): by stall
samples, with shared-memory wavefronts (ideal vs actual) per instruction.

    python tools/ncu_src.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                      "regex:" + kern], capture_output=True, text=True).stdout
lines = out.splitlines()
rows = [r for r in csv.DictReader(io.StringIO("\n".join(lines[1:])))
        if (r.get("Warp Stall Sampling (All Samples)") or "0").isdigit()]  # one block per matching kernel
tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
print(f"{len(rows)} SASS lines, {tot} stall samples")
key = lambda r: int(r["Warp Stall Sampling (All Samples)"] or 0)
for r in sorted(rows, key=key, reverse=True)[:top]:
    wf, wi = r.get("L1 Wavefronts Shared", "0"), r.get("L1 Wavefronts Shared Ideal", "0")
    print(f"{key(r):7d} {100.0 * key(r) / max(tot, 1):5.1f}%  exec {r['Instructions Executed']:>9s}  "
          f"smem wf {wf:>8s}/{wi:>8s}  {r['Address'][-5:]}  {r['Source'].strip()[:70]}")
