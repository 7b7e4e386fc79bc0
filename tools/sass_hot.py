"""Top stalled SASS instructions of an ncu report's source page.

    python tools/sass_hot.py gpurun_out/x.ncu-rep [kernel-regex] [N]
"""
import csv
import io
import subprocess
import sys


def main(path, kregex=None, n=30):
    cmd = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"]
    if kregex:
        cmd += ["-k", f"regex:{kregex}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    lines = out.splitlines()
    blocks, cur = [], None
    for ln in lines:
        if ln.startswith('"Kernel Name"'):
            cur = [ln]
            blocks.append(cur)
        elif cur is not None:
            cur.append(ln)
    for b in blocks[:1]:
        print(b[0][:160])
        rows = list(csv.reader(io.StringIO("\n".join(b[1:]))))
        h = rows[0]
        ia, isrc = h.index("Address"), h.index("Source")
        ist = h.index("Warp Stall Sampling (All Samples)")
        iex = h.index("Instructions Executed")
        data = []
        for r in rows[1:]:
            try:
                data.append((int(r[ist]), r[ia][-5:], r[isrc].strip(), r[iex]))
            except (ValueError, IndexError):
                pass
        tot = sum(d[0] for d in data) or 1
        print(f"total samples {tot}")
        for s, a, src, ex in sorted(data, reverse=True)[:n]:
            print(f"{100 * s / tot:5.1f}% {a} {ex:>8} {src[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None,
         int(sys.argv[3]) if len(sys.argv) > 3 else 30)
