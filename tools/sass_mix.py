"""Executed-instruction mix (by opcode) of one kernel in an ncu report.

    python tools/sass_mix.py gpurun_out/x.ncu-rep kernel-regex [N]
"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main(path, kregex, n=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "sass", "-k", f"regex:{kregex}"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = [i for i, ln in enumerate(lines) if ln.startswith('"Kernel Name"')]
    block = lines[start[0] + 1:start[1]] if len(start) > 1 else lines[start[0] + 1:]
    rows = list(csv.reader(io.StringIO("\n".join(block))))
    h = rows[0]
    isrc, iex = h.index("Source"), h.index("Instructions Executed")
    mix = Counter()
    for r in rows[1:]:
        if len(r) <= iex:
            continue
        try:
            ex = int(r[iex])
        except ValueError:
            continue
        op = r[isrc].strip().lstrip("@!P0123456789UPT ").split(" ")[0].split(".")[0]
        mix[op] += ex
    tot = sum(mix.values())
    print(f"total warp instructions {tot}")
    for op, c in mix.most_common(n):
        print(f"{100 * c / tot:5.1f}% {c:12d} {op}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
