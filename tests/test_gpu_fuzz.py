"""Randomised parity sweep (tools/fuzz_parity.py): random problems --
stencil shapes and CSR matrices x methods x shifts x preconditioners x x0 x
gaps -- device vs oracle in the device's reduction order, bit for bit
(breakdowns included)."""

import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


@pytest.mark.gpu
@pytest.mark.parametrize("mode,seed", [("tree", 11), ("tree", 12), ("reference", 13), ("dist", 9), ("dist", 14)])
def test_random_problems_bitwise(mode, seed):
    """tree: device vs oracle in the device order; reference: device in the
    reference order vs the oracle's blocked_dot; dist: 2-8 virtual ranks
    through the peer exchange vs one GPU."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import fuzz_parity
    assert fuzz_parity.run(20 if mode != "dist" else 40, seed, log=lambda *a: None, mode=mode) == []
