"""Out-of-bounds and uninitialised-memory checks without compute-sanitizer (needs a B200).

compute-sanitizer is closed on this GPU pool (profiles/r02_sanitize.txt), so
VERDICT r01 item 4's memcheck / initcheck is done with guard bands instead:
every solver vector and the workspace are views into arenas whose padding
(and, for the workspace, whose whole body) is filled with a poison pattern.
After each solve

* every guard band must still hold the poison -- no kernel wrote outside its
  vector or its workspace (memcheck, writes);
* the result must be bit-identical to the same solve with a DIFFERENT poison
  pattern and to the normal allocation -- no result depends on memory outside
  the vectors or on workspace bytes nobody initialised (memcheck reads /
  initcheck).

Every kernel family runs: TMA 3D and 2D sweeps, the register sweep, the
persistent small-problem solver, the split CSR path (window and pipelined
SpMV), the window and the column-sorted SpMV, IC(0), p-CG-rr replacement, gap
instrumentation, classic CG and the reference reduction order.
"""

import os

import numpy as np
import pytest

import paper_1706_05988_b200 as K
from paper_1706_05988_b200 import problems
from paper_1706_05988_b200.solvers import _Solve

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

PAD = 4096                                  # elements of guard band on each side


class Arena:
    """Hands out views with poisoned guard bands; remembers them for the check."""

    def __init__(self, word):
        self.word = word                     # 64-bit poison pattern
        self.blocks = []

    def __call__(self, count, dtype):
        esz = torch.empty(0, dtype=dtype).element_size()
        nbytes = count * esz
        raw = torch.empty((nbytes + 2 * PAD * 8 + 7) // 8, dtype=torch.int64, device="cuda")
        raw.fill_(self.word)
        body = raw.view(torch.uint8)[PAD * 8:PAD * 8 + nbytes]
        self.blocks.append((raw, nbytes))
        return body.view(dtype)

    def check(self):
        for raw, nbytes in self.blocks:
            u8 = raw.view(torch.uint8)
            lo = u8[:PAD * 8].view(torch.int64)
            hi = u8[PAD * 8 + nbytes:PAD * 8 + nbytes + PAD * 8]
            ref = torch.full((1,), self.word, dtype=torch.int64, device="cuda").view(torch.uint8)
            assert bool((lo == self.word).all()), "write below a vector / the workspace"
            pat = ref.repeat((hi.numel() + 7) // 8)
            off = (PAD * 8 + nbytes) % 8        # the band after the body starts mid-word
            assert bool((hi == torch.roll(pat, -off)[:hi.numel()]).all()), "write past a vector / the workspace"


POISONS = [0x7FF4DEADBEEF0001, -0x0123456789ABCDEF]     # a signalling NaN and a large negative pattern


def rows(res):
    return [(r.iter, r.alpha, r.beta, r.gamma, r.delta, r.rnorm_recursive, r.rnorm_true, r.gap_f)
            for r in res.history]


CASES = [
    ("tma3d", lambda: (K.Stencil3D(64, 24, 16), None), dict(method="pcg_sh", shift=1.0), {"persistent": False}),
    ("tma2d_jacobi", lambda: (K.Stencil2D(1024, 30), "jacobi"), dict(method="pcg_sh", shift=0.4), {"persistent": False}),
    ("register", lambda: (K.Stencil3D(33, 9, 20), None), dict(method="pcg_rr"), {}),
    ("persistent", lambda: (K.Stencil2D(60, 50), None), dict(method="pcg_sh", shift=2.0), {}),
    ("csr_window", lambda: (problems.varcoef_3d(11, seed=1), "jacobi"), dict(method="pcg_sh", shift=0.5), {}),
    ("csr_pipe", lambda: (problems.banded_spd(20_000, seed=2, band=3000), "jacobi"), dict(method="pcg_rr"),
     {"env": ("KPL_CSR_GATHER", "csr")}),
    ("csr_band", lambda: (problems.banded_spd(20_001, seed=2, band=3000), "jacobi"), dict(method="pcg_rr"),
     {"env": ("KPL_CSR_GATHER", "band"), "env2": ("KPL_BAND_W", "1022")}),
    ("csr_sorted", lambda: (problems.banded_spd(20_000, seed=2, band=3000), "jacobi"),
     dict(method="pcg_sh", shift=0.4), {"env": ("KPL_CSR_GATHER", "sorted")}),
    ("csr_sorted_pcg", lambda: (problems.banded_spd(20_000, seed=2, band=3000), "jacobi"),
     dict(method="pcg", shift=0.0), {"env": ("KPL_CSR_GATHER", "sorted")}),
    ("ic0", lambda: (K.laplacian_2d(30, 20), "ic0"), dict(method="pcg_sh", shift=0.3), {}),
    ("gaps", lambda: (K.Stencil2D(50, 40), None), dict(method="pcg_sh", shift=1.0, track_gaps=True), {}),
    ("cg", lambda: (K.laplacian_2d(70, 50), "jacobi"), dict(method="cg"), {}),
    ("reference_order", lambda: (K.laplacian_2d(40, 30), None), dict(method="pcg_sh", shift=1.0), {"order": 1}),
]


@pytest.mark.parametrize("name,make,kw,opt", CASES, ids=[c[0] for c in CASES])
def test_guard_bands_and_no_uninitialised_reads(monkeypatch, name, make, kw, opt):
    for key in ("env", "env2"):
        if key in opt:
            monkeypatch.setenv(*opt[key])
    A, mk = make()
    M = {"jacobi": K.make_jacobi, "ic0": K.make_ic0}.get(mk, lambda A: None)(A)
    b = np.random.default_rng(4).standard_normal(A.n)
    cfg = K.SolverConfig(max_iters=60, rtol=1e-10, **kw)
    order = "reference" if opt.get("order") else "tree"
    with K.reduction_order(order):
        want = _Solve(A, M, b, None, cfg, persistent=opt.get("persistent")).run()
        for word in POISONS:
            arena = Arena(word)
            got = _Solve(A, M, b, None, cfg, persistent=opt.get("persistent"), alloc=arena).run()
            torch.cuda.synchronize()
            arena.check()
            assert rows(got) == rows(want), (name, hex(word))
            assert np.asarray(got.x).tobytes() == np.asarray(want.x).tobytes(), (name, hex(word))
            assert got.replacements == want.replacements
