"""Run the resident-key tensor-core attention at the C2 triangle shape
(nb=256, L=256, H=8, D=32, transposed bias) once: a profiling target."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2211_00235_b200 import kernels as K  # noqa: E402
from test_gpu_attention import run_case  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "transposed"
run_case(K, 256, 256, 8, 32, True, mode, dtype=torch.bfloat16)
torch.cuda.synchronize()
