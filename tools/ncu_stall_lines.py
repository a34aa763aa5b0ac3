"""Warp-stall samples of one kernel in an ncu report, summed per source line.

    python tools/ncu_stall_lines.py gpurun_out/r1e_c2_tc.ncu-rep paper_2511_22333_b200/libpatb200.so \\
        _ZN3pat3tc214fwd_tc2_kernelILi128E13__nv_bfloat16 [top]

Reads the SASS source page (`ncu -i --page source --csv --print-source sass`),
maps each instruction offset to file:line with `nvdisasm -g` of the same build
(compiled with -lineinfo) and prints the top lines by share of all samples."""

import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main(rep, lib, fn_prefix, top=25):
    page = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(page)))
    hdr = rows[1]
    data = rows[2:]
    ia, iss = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
    base = int(data[0][ia], 16)
    tot = sum(float(r[iss] or 0) for r in data) or 1.0
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True, check=True)
        sass = ""
        for f in sorted(os.listdir(d)):
            if f.endswith(".cubin"):
                sass += subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, f)], capture_output=True,
                                       text=True).stdout
    lines = sass.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith(".text." + fn_prefix))
    cur, m = None, {}
    for l in lines[start + 1:]:
        if l.startswith(".text."):
            break
        mm = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if mm:
            cur = f"{os.path.basename(mm.group(1))}:{mm.group(2)}"
        a = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if a:
            m[int(a.group(1), 16)] = cur
    if len(m) != len(data):
        print(f"warning: {len(data)} profiled instructions vs {len(m)} in {lib} (different build?)")
    per = {}
    for r in data:
        k = m.get(int(r[ia], 16) - base)
        per[k] = per.get(k, 0.0) + float(r[iss] or 0)
    for k, v in sorted(per.items(), key=lambda x: -x[1])[:top]:
        print(f"{100 * v / tot:5.1f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 25)
