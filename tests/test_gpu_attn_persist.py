"""The persistent short-sequence kernel (attn_persist.cu; the default for non-causal N <= 2048: the non-causal cases of
tests/attn_kernel_check.py up to 2100 tokens) and the same cases with it switched off (SAGE3_PERSIST=0), each against
the oracle in its own process."""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.gpu
@pytest.mark.parametrize("persist", ["0", "1"])
def test_attention_persistent_selection_parity(persist):
    env = dict(os.environ, SAGE3_PERSIST=persist, SAGE3_ATTN_KERNEL="2")
    p = subprocess.run([sys.executable, os.path.join(HERE, "attn_kernel_check.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    assert p.returncode == 0 and "ALL OK" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]
