"""GPU: the reference's own acceptance gate (proj/tests/acceptance.cpp,
criteria 1-7), compiled unchanged and linked against the B200 drop-in
libchainhull.so (build/acceptance_b200, built by `make` where
/root/reference exists and shipped prebuilt to the GPU box)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "build", "acceptance_b200")


@pytest.mark.parametrize("criterion", [1, 2, 3, 4, 5, 6, 7])
def test_reference_acceptance_criterion(criterion):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(BIN):
        pytest.skip("build/acceptance_b200 not built (needs /root/reference at build time)")
    p = subprocess.run([BIN, str(criterion)], capture_output=True, text=True, timeout=600)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "[PASS]" in p.stdout
