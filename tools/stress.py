"""Repeat the training step many times to catch intermittent hangs.

    python tools/stress.py --steps 2000 [--eager]   (CUDA_LAUNCH_BLOCKING=1 with
    --eager pins a hang to the launching wrapper: faulthandler dumps the
    Python stack after --timeout seconds without progress)
"""

import argparse
import faulthandler
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--eager", action="store_true")
    ap.add_argument("--timeout", type=float, default=30.0)
    ap.add_argument("--config", default="af2")
    a = ap.parse_args()
    import paper_2211_00235_b200 as pkg
    from paper_2211_00235_b200 import schedules as S
    from bench import CONFIGS
    dev = torch.device("cuda", 0)
    cfg = pkg.EvoConfig(**CONFIGS[a.config])
    store = pkg.init_params(cfg, 32, device=dev)
    st = S.StepState(cfg, store, "bf16", dev)
    st.pack()
    m_h, z_h = S.make_batch(cfg, 32, 1, device="cpu")[0]
    m, z = m_h.to(dev), z_h.to(dev)
    for _ in range(3):
        S.full_step(st, m, z)
    torch.cuda.synchronize()
    if a.eager:
        fn = lambda: S.full_step(st, m, z)  # noqa: E731
    else:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            S.full_step(st, m, z)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            S.full_step(st, m, z)
        fn = g.replay
    t0 = time.time()
    for i in range(a.steps):
        faulthandler.dump_traceback_later(a.timeout, exit=True)
        fn()
        if i % 10 == 9:
            torch.cuda.synchronize()
        if i % 200 == 199:
            print(f"step {i + 1} ok ({time.time() - t0:.1f} s)", flush=True)
    torch.cuda.synchronize()
    faulthandler.cancel_dump_traceback_later()
    print(f"done {a.steps} steps in {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main()
