"""Top SASS instructions by warp-stall samples for one kernel of an ncu report.

  python tools/ncu_hot.py report.ncu-rep kernel_regex [n]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = [r for r in rows[2:] if r and r[0].startswith("0x")]
if len(data) % 2 == 0 and data and data[0][0] == data[len(data) // 2][0]:
    data = data[:len(data) // 2]
si, ii = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
f = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
tot, toti = sum(f(r[si]) for r in data), sum(f(r[ii]) for r in data)
print(f"{len(data)} instructions, {tot:.0f} samples, {toti:.0f} executed")
for k in sorted(sorted(range(len(data)), key=lambda k: -f(data[k][si]))[:n]):
    r = data[k]
    print(f"{k:5d} {100 * f(r[si]) / tot:5.1f}% {100 * f(r[ii]) / toti:5.1f}%  {r[1][:80]}")
