"""Hot source lines of one kernel from an ncu report (--import-source captures):
warp-stall samples per CUDA source line.

  python tools/ncu_src_hot.py REPORT.ncu-rep KERNEL_REGEX [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}", "--launch-skip",
                      skip, "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = [k for k, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r][0]
i_s = rows[hi].index("Warp Stall Sampling (All Samples)")
out, tot = [], 0
for r in rows[hi + 1:]:
    if len(r) <= i_s or not r[0]:
        continue  # SASS rows have an empty line number
    try:
        v = int(r[i_s])
    except ValueError:
        continue
    tot += v
    out.append((v, r[0], r[1][:100]))
out.sort(reverse=True)
print(f"{kern}: {tot} warp-stall samples")
for v, ln, src in out[:top]:
    print(f"{v:7d} {100.0 * v / max(tot, 1):5.1f}%  line {ln}: {src}")
