"""Run the streamed-key attention at crop r = 384 shapes (profiling target):
triangle-end (transposed bias) and the same shape without a bias."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2211_00235_b200 import kernels as K  # noqa: E402
from test_gpu_attention import run_case  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "transposed"
run_case(K, 384, 384, 8, 32, True, mode, dtype=torch.bfloat16)
torch.cuda.synchronize()
