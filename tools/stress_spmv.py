"""Repeat-and-compare stress of the CSR SpMV layouts (KPL_CSR_GATHER = band | sorted | csr): every launch must
equal the oracle bit for bit, with another stream keeping the GPU busy (this is how the r2 race in the bulk-TMA
variant of the column-sorted kernel was found; that kernel was removed).

    python tools/stress_spmv.py [band,sorted,csr] [reps]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1706_05988_b200 as K
from paper_1706_05988_b200 import problems, device as D
from oracle import kpl_oracle as O

def fresh(A):
    return K.SparseMatrix(A.n, A.row_ptr.copy(), A.col_idx.copy(), A.values.copy())

side = torch.cuda.Stream()
junk = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
for name, A in [("band_wide", problems.banded_spd(70_001, seed=1)), ("band", problems.banded_spd(30_000, seed=3, band=8000)),
                ("big", problems.banded_spd(400_000, seed=2))]:
    v = np.random.default_rng(7).standard_normal(A.n); v[::5] = 0.0; v[1::7] = -0.0
    want = O.spmv(O.as_oracle_operator(A), v)
    vd = torch.as_tensor(v, device="cuda")
    for mode in (sys.argv[1].split(",") if len(sys.argv) > 1 else ("band", "sorted", "csr")):
        os.environ["KPL_CSR_GATHER"] = mode
        bad = 0
        for rebuild in range(6):
            B = fresh(A)
            for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 150):
                if rep % 3 == 0:
                    with torch.cuda.stream(side):
                        junk.normal_()            # concurrent HBM traffic and SM occupancy
                got = K.spmv(B, vd)
                if rep % 10 == 0 or True:
                    g = got.cpu().numpy()
                    if g.tobytes() != want.tobytes():
                        bad += 1
                        d = np.nonzero(g.view(np.int64) != want.view(np.int64))[0]
                        print("MISMATCH", name, mode, rebuild, rep, len(d), d[:5], g[d[:3]], want[d[:3]], flush=True)
        print(name, mode, "mismatches:", bad, flush=True)
torch.cuda.synchronize()
