import sys, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2211_00235_b200 import kernels as K
from test_gpu_attention import run_case
run_case(K, 384, 384, 8, 32, True, "transposed", dtype=torch.bfloat16)
torch.cuda.synchronize()
