"""Every backward pair kernel the library can select (FPDT_BWD_KERNEL, read once per process) against the oracle:
the default routing is covered by the other GPU tests; here the forced variants run the bf16 parity cases of
test_gpu_parity.py in a child process:
  q64  attn_bwd_q64_kernel at d = 64 / 80 / 128 (default only at 128)
  v2   attn_bwd_kernel (vector-atomic dQ) at d = 64 / 80 / 128
  pipe attn_bwd_pipe_kernel at d = 64 / 80 (its only head_dims)"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("kernel,select", [("q64", "bf16"), ("v2", "bf16"), ("pipe", "config1_bf16 or (bf16_shapes and not 128)")])
def test_forced_backward_kernel(kernel, select):
    env = dict(os.environ, FPDT_BWD_KERNEL=kernel)
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-q", "-x",
                        "-p", "no:cacheprovider", "-k", select], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
