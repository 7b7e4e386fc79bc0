"""Per-launch breakdown of one train step: run under ncu's launch list, then
join the GEMM / attention launches with their shapes.

    ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none \
        --profile-from-start off --csv --log-file gpurun_out/trace.csv \
        python tools/step_trace.py --shapes gpurun_out/trace_shapes.json
    python tools/step_trace.py --join gpurun_out/trace.csv gpurun_out/trace_shapes.json

Only the one eager step between cudaProfilerStart/Stop is profiled.
"""

import argparse
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(args):
    import torch

    import paper_2211_00235_b200 as pkg
    from bench import CONFIGS
    from paper_2211_00235_b200 import kernels as K, schedules as S

    dev = torch.device("cuda", 0)
    kw = dict(CONFIGS[args.config])
    if args.crop:
        kw["r"] = args.crop
    cfg = pkg.EvoConfig(**kw)
    store = pkg.init_params(cfg, 32, device=dev)
    st = S.StepState(cfg, store, args.precision, dev)
    st.pack()
    m, z = S.make_batch(cfg, 32, 1, device=dev)[0]
    for _ in range(3):
        S.full_step(st, m, z)
    torch.cuda.synchronize()
    prof, shapes = [], []
    K.PROFILE, K.PROFILE_SHAPES = prof, shapes
    torch.cuda.profiler.start()
    S.full_step(st, m, z)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    K.PROFILE = K.PROFILE_SHAPES = None
    out = [[fam, fl, list(shp) if shp else None] for (fam, fl, _, _), shp in zip(prof, shapes)]
    with open(args.shapes, "w") as f:
        json.dump(out, f)


def family_of(name):
    if "gemm_tc_kernel" in name or "gemm_simt_kernel" in name or "skinny_" in name:
        return "gemm"
    if "attn_fwd" in name or "attn_flash_fwd" in name:
        return "attention_fwd"
    if "attn_bwd_prep" in name or "long_prep" in name:
        return "attention_bwd"
    return None


def join(csv_path, shapes_path, json_out=None):
    with open(shapes_path) as f:
        calls = json.load(f)
    rows = []
    dram = {}  # launch id -> bytes (when the dram metrics were collected)
    with open(csv_path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        name = r.get("Metric Name")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        if name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            dram[r["ID"]] = dram.get(r["ID"], 0.0) + v * scale
            continue
        if name != "gpu__time_duration.sum":
            continue
        us = v / 1e3 if unit.startswith("n") else (v if unit.startswith("u") else v * 1e3)
        rows.append((r["Kernel Name"], us, r["ID"]))
    # attach each family-starting launch to the next call of that family
    queues = {}
    for fam, fl, shp in calls:
        queues.setdefault(fam, []).append((fl, shp))
    cur = None
    groups = []
    for name, us, lid in rows:
        fam = family_of(name)
        if fam is not None and queues.get(fam):
            fl, shp = queues[fam].pop(0)
            cur = [fam, shp, fl, 0.0, [], 0.0]
            groups.append(cur)
        elif fam is not None or cur is None or not (
                (cur[0] == "gemm" and ("splitk_reduce" in name or "skinny_reduce" in name)) or
                (cur[0] == "attention_bwd" and ("attn_bwd" in name or "attn_flash" in name
                                                or "reduce_lead" in name
                                                or "colsum_stage2" in name))):
            cur = [name.split("(")[0][:48], None, 0.0, 0.0, [], 0.0]
            groups.append(cur)
        cur[3] += us
        cur[4].append(name.split("(")[0].split("<")[0][-28:])
        cur[5] += dram.get(lid, 0.0)
    total = sum(g[3] for g in groups)
    fam_tot = {}
    for g in groups:
        if g[0] in ("gemm", "attention_fwd", "attention_bwd"):
            f = fam_tot.setdefault(g[0], [0.0, 0.0, 0, 0.0])
            f[0] += g[3]
            f[1] += g[2]
            f[2] += 1
            f[3] += g[5]
    for k, (us, fl, n, byt) in fam_tot.items():
        print(f"family {k}: {n} launches, {us:.1f} us, {fl / us / 1e6:.1f} TF/s, "
              f"DRAM {byt / 1e6:.1f} MB ({byt / max(n, 1) / 1e6:.2f} MB per launch)")
    if json_out:
        with open(json_out, "w") as f:
            json.dump({"source": os.path.basename(csv_path),
                       "families": {k: {"launches": n, "us": us, "dram_bytes": byt,
                                        "dram_bytes_per_launch": byt / max(n, 1)}
                                    for k, (us, fl, n, byt) in fam_tot.items()}}, f, indent=1)
    agg = {}
    for fam, shp, fl, us, names, _b in groups:
        key = f"{fam} {shp}" if shp else fam
        a = agg.setdefault(key, [0.0, 0.0, 0])
        a[0] += us
        a[1] += fl
        a[2] += 1
    print(f"total {total:.1f} us over {len(rows)} launches")
    for key, (us, fl, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        tf = fl / us / 1e6 if fl else 0.0
        print(f"{us:9.1f} us {100 * us / total:5.1f}% {n:3d}x {tf:7.1f} TF/s  {key}")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="af2")
    ap.add_argument("--precision", default="bf16")
    ap.add_argument("--crop", type=int, default=0)
    ap.add_argument("--shapes", default="gpurun_out/trace_shapes.json")
    ap.add_argument("--join", nargs=2, metavar=("CSV", "SHAPES"))
    ap.add_argument("--family-json", default=None,
                    help="with --join: write per-family DRAM bytes per launch here")
    a = ap.parse_args()
    if a.join:
        join(*a.join, json_out=a.family_json)
    else:
        run(a)
