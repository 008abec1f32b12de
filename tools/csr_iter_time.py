"""Device time of N p-CG-sh iteration sweeps (no result check) -- A/B timing helper.

    KPL_CSR_GATHER=auto|band|csr|sorted [KPL_LONG=1] python tools/csr_iter_time.py [c2c,c4,c5] [chunk_blocks]

Matrices are cached under /tmp/kpl_cache (generation of config 5 takes ~30 s).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_05988_b200 as K  # noqa: E402
from paper_1706_05988_b200 import problems  # noqa: E402
from paper_1706_05988_b200.solvers import _Solve  # noqa: E402

CACHE = "/tmp/kpl_cache"
GEN = {
    "c2c": lambda: K.laplacian_2d(2048, 2048),
    "c4": lambda: problems.varcoef_3d(256, seed=0, check_symmetry=False),
    "c5": lambda: problems.banded_spd(2_000_000, seed=0),
}
RHS = {
    "c2c": lambda n: np.random.default_rng(0).random(n),
    "c4": lambda n: np.random.default_rng(1).standard_normal(n),
    "c5": lambda n: np.random.default_rng(1).standard_normal(n),
}


def matrix(name):
    os.makedirs(CACHE, exist_ok=True)
    f = os.path.join(CACHE, name + ".npz")
    if os.path.exists(f):
        d = np.load(f)
        return K.SparseMatrix(int(d["n"]), d["row_ptr"], d["col_idx"], d["values"], check_symmetry=False)
    A = GEN[name]()
    np.savez(f, n=A.n, row_ptr=A.row_ptr, col_idx=A.col_idx, values=A.values)
    return A


def main():
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2c", "c4", "c5"]
    cb = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    tag = (f"gather={os.environ.get('KPL_CSR_GATHER', 'auto')} nt={os.environ.get('KPL_SORTED_NT', '512')} "
           f"chunk_blocks={cb or 'default'}")
    for name in names:
        A = matrix(name)
        M = K.make_jacobi(A)
        b = torch.as_tensor(RHS[name](A.n), device="cuda")
        S = _Solve(A, M, b, None, K.SolverConfig(method="pcg_sh", shift=0.4, max_iters=100), chunk_blocks=cb)
        S.init()
        S.iterate(1)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            S.iterate(9)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 9)
            S = _Solve(A, M, b, None, K.SolverConfig(method="pcg_sh", shift=0.4, max_iters=100), chunk_blocks=cb)
            S.init()
            S.iterate(1)
            torch.cuda.synchronize()
        print(name, tag, f"{best:.4f} ms/iteration (best of 3 x 9)", flush=True)
        if os.environ.get("KPL_LONG"):
            # sustained: 400 iterations with the true-residual cadence, one enqueue
            S = _Solve(A, M, b, None, K.SolverConfig(method="pcg_sh", shift=0.4, max_iters=1000), chunk_blocks=cb)
            S.init()
            S.iterate(10)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            S.iterate(400)
            e1.record()
            torch.cuda.synchronize()
            print(name, tag, f"{e0.elapsed_time(e1) / 400:.4f} ms/iteration sustained (400 iterations incl. cadence)",
                  flush=True)


if __name__ == "__main__":
    main()
