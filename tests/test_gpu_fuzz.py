"""Randomised parity sweep (tools/fuzz_parity.py): 40 random problems --
stencil shapes and CSR matrices x methods x shifts x preconditioners x x0 x
gaps -- device vs oracle in the device's reduction order, bit for bit
(breakdowns included)."""

import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [11, 12])
def test_random_problems_bitwise(seed):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import fuzz_parity
    assert fuzz_parity.run(20, seed, log=lambda *a: None) == []
