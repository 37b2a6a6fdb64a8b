"""Executed-instruction mix (by SASS opcode) of one kernel of an ncu report.

  python tools/ncu_opmix.py report.ncu-rep kernel_regex [n]
"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = [r for r in rows[2:] if r and r[0].startswith("0x")]
if len(data) % 2 == 0 and data and data[0][0] == data[len(data) // 2][0]:
    data = data[:len(data) // 2]
ii = h.index("Instructions Executed")
f = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
mix = collections.Counter()
for r in data:
    toks = r[1].split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    mix[op.split(".")[0]] += f(r[ii])
tot = sum(mix.values())
print(f"{tot:.0f} warp instructions executed")
for op, c in mix.most_common(n):
    print(f"{op:12s} {c:14.0f} {100 * c / tot:6.2f}%")
