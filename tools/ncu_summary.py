"""One-line-per-kernel summary of an ncu --set full report: duration,
issue activity, tensor-pipe activity, DRAM throughput / bytes, top stalls.

    python tools/ncu_summary.py report.ncu-rep [report2 ...]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "us"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor%"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("dram__bytes_read.sum", "dramR"),
    ("dram__bytes_write.sum", "dramW"),
    ("launch__registers_per_thread", "regs"),
]


def col(h, key):
    """Index of the column named `key` (the raw page may prefix a section)."""
    for i, name in enumerate(h):
        if name == key or name.endswith("." + key):
            return i
    return None


def main(paths):
    for path in paths:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            continue
        h, units = rows[0], rows[1]
        print(f"# {path}")
        for r in rows[2:]:
            name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")[:60]
            parts = []
            for k, lab in KEYS:
                i = col(h, k)
                if i is not None and r[i]:
                    unit = units[i] if lab.startswith("dram") and not lab.endswith("%") else ""
                    parts.append(f"{lab}={r[i]}{unit}")
            st = []
            for k in h:
                if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                    try:
                        st.append((float(r[h.index(k)].replace(",", "")), k[33:]))
                    except ValueError:
                        pass
            tot = sum(v for v, _ in st) or 1.0
            st.sort(reverse=True)
            stalls = ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in st[:3])
            print(f"{name}\n    " + "  ".join(parts) + f"\n    stalls: {stalls}")


if __name__ == "__main__":
    main(sys.argv[1:])
