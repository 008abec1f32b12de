"""IC(0) timing on the device: factor (one sync-free sweep) and apply (two
substitution sweeps), CUDA events, beside the CPU oracle's apply (C, 1 core)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1706_05988_b200 as K
from paper_1706_05988_b200 import problems
from oracle import kpl_oracle as O


def main():
    out = []
    for name, A in (("lapl512", K.laplacian_2d(512, 512)), ("lapl2048", K.laplacian_2d(2048, 2048)),
                    ("varcoef64", problems.varcoef_3d(64, seed=0))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        M = K.make_ic0(A)
        torch.cuda.synchronize()
        t_factor = time.perf_counter() - t0
        v = torch.randn(A.n, dtype=torch.float64, device="cuda")
        for _ in range(3):
            M.apply(v)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            M.apply(v)
        e1.record()
        torch.cuda.synchronize()
        t_apply = e0.elapsed_time(e1) / reps
        oM = O.as_oracle_precond(M)
        hv = v.cpu().numpy()
        t0 = time.perf_counter()
        ref = oM.apply(hv)
        t_cpu = (time.perf_counter() - t0) * 1e3
        same = ref.tobytes() == M.apply(hv).tobytes()
        nnz = len(M._l[1])
        rec = {"case": name, "n": A.n, "nnz_L": nnz, "factor_s_incl_host_setup": round(t_factor, 4),
               "apply_ms": round(t_apply, 4), "cpu_oracle_apply_ms": round(t_cpu, 3), "bitwise_vs_oracle": same,
               "note": "apply_ms includes the workspace alloc + flag reset of the API call"}
        print(json.dumps(rec), flush=True)
        out.append(rec)


if __name__ == "__main__":
    main()
