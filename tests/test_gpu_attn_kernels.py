"""Both attention kernels of the north_star path (attn.cu: two softmax warpgroups, the d = 128 default; attn3.cu:
three softmax warpgroups, the d = 64 default) against the oracle, each forced for a whole process with
SAGE3_ATTN_KERNEL, so the kernel that is not the default for a d is still parity-tested; plus attn.cu with K/V tiles
shared by 2-CTA clusters through TMA multicast (SAGE3_KV_MULTICAST=1; non-causal cases with an even tile count)."""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", ["2", "3", "2mc"])
def test_attention_kernel_selection_parity(kernel):
    env = dict(os.environ, SAGE3_ATTN_KERNEL=kernel[0], SAGE3_KV_MULTICAST="1" if kernel.endswith("mc") else "0")
    p = subprocess.run([sys.executable, os.path.join(HERE, "attn_kernel_check.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    assert p.returncode == 0 and "ALL OK" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]
