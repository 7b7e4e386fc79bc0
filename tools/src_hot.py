"""Per-source-line warp-stall samples of one kernel in an ncu report.

    python tools/src_hot.py gpurun_out/x.ncu-rep kernel-regex [N]
"""
import csv
import io
import subprocess
import sys


def main(path, kregex, n=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "cuda,sass", "-k", f"regex:{kregex}"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    data, ist, fname = [], None, "?"
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            ist = r.index("Warp Stall Sampling (All Samples)")
            continue
        if ist is None or len(r) <= ist or not r[0]:
            continue
        try:
            data.append((int(r[ist]), f"{fname}:{r[0]}", r[1].strip()[:100]))
        except ValueError:
            pass
    tot = sum(d[0] for d in data) or 1
    print(f"total samples {tot}")
    for s, ln, src in sorted(data, reverse=True)[:n]:
        print(f"{100 * s / tot:5.1f}% {ln:>22} {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
