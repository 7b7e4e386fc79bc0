"""Run the streamed-key attention once at a chosen shape (profiling target).

    python tools/flash_prof.py [mode] [shape]
mode: transposed | plain | none;  shape: tri384 (nb=384, L=384, H=8, D=32),
col1024d8 (the C3 extra-MSA column attention: nb=256, L=1024, H=8, D=8),
row256d8 (C3 extra-MSA row attention: nb=1024, L=256, H=8, D=8)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2211_00235_b200 import kernels as K  # noqa: E402
from test_gpu_attention import run_case  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "transposed"
shape = sys.argv[2] if len(sys.argv) > 2 else "tri384"
nb, L, H, D, seq = {"tri384": (384, 384, 8, 32, True), "col1024d8": (256, 1024, 8, 8, True),
                    "row256d8": (1024, 256, 8, 8, False)}[shape]
run_case(K, nb, L, H, D, seq, mode, dtype=torch.bfloat16)
torch.cuda.synchronize()
