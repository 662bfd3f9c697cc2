"""One cuBLAS DGEMM (torch.matmul float64, 8192^3): the FP64 tensor-pipe
reference an ncu capture of k_gemm is compared with."""
import torch

a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
torch.matmul(a, b)
torch.cuda.synchronize()
