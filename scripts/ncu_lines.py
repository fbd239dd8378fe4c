"""Aggregate an ncu source-page capture (SASS warp-stall samples) by CUDA
source line, using nvdisasm -g line info of the same library build.
Development aid:  python scripts/ncu_lines.py REPORT.ncu-rep KERNEL_SUBSTRING [N]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
lib = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_1110_6220_b200", "libeikonal_b200.so")
csvtxt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                        capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(csvtxt)))
hdr, data = rows[1], rows[2:]
iss = hdr.index("Warp Stall Sampling (All Samples)")
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=d, capture_output=True)
    instrs = []
    for f in sorted(os.listdir(d)):
        txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, f)], capture_output=True,
                             text=True).stdout
        infn, cur = False, None
        for L in txt.split("\n"):
            if ".section" in L and ".text." in L:
                infn = kname in L
                continue
            if not infn:
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', L)
            if m:
                cur = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", L)
            if m:
                instrs.append(cur)
        if instrs:
            break
assert len(instrs) == len(data), (len(instrs), len(data))
agg = collections.Counter()
for k, r in enumerate(data):
    if r[iss].isdigit():
        agg[instrs[k]] += int(r[iss])
tot = sum(agg.values())
print("samples", tot)
for key, s in agg.most_common(top):
    print(f"{s:8d} {100 * s / tot:5.1f}%  {key[0]}:{key[1]}")
