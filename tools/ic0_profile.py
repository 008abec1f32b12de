"""Target for ncu: IC(0) factor + a few applies on lapl:512x512."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1706_05988_b200 as K  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
A = K.laplacian_2d(n, n)
M = K.make_ic0(A)
v = torch.randn(A.n, dtype=torch.float64, device="cuda")
for _ in range(3):
    M.apply(v)
torch.cuda.synchronize()
print("ok")
