"""Every row of every output at BASELINE.json configs[1]'s full shape, against an exact closed form (SURVEY §8(c) c.3
"class keys", c.5 (iii) "a class-keys run at the same shape on all tensors").

Inputs: the "class" distribution (fpdt_inputs: keys take one of K = 4 class vectors, a large-norm class only in the
second half of the sequence, so the running max jumps at chunk boundaries), S = 524,288, 32 heads, head_dim 80,
chunk 65,536, bf16, offload on, world size 1: the bench's launch configuration.  For class keys the attention and its
gradient have a closed form computable in O(S K d^2) (oracle/closed_forms.py, pinned against the plain definition in
tests/test_oracle.py), so O, lse, dQ, dK and dV of EVERY row are compared for one head (the other heads run the same
arithmetic and are covered by the sampled-row tests).  Bar: normwise max relative error <= 1e-2 (north_star, bf16)."""
import ctypes

import numpy as np
import pytest
import torch

import fpdt_inputs as gen
from fpdt_testlib import TOL, rel_err
from oracle import closed_forms

pytestmark = pytest.mark.gpu

S, H, D, C = 524288, 32, 80, 65536
HEAD = 31


def test_fullsize_class_keys_all_rows():
    from paper_2408_16978_b200 import _lib, fpdt
    torch.cuda.set_device(0)
    genlib = _lib.load_generator()

    def gen_tensor(name):
        t = torch.empty(S, H, D, dtype=torch.bfloat16, device="cuda")
        rc = genlib.fpdt_gen_fill(ctypes.c_void_p(t.data_ptr()), 0, gen.TENSOR_IDS[name], gen.DIST_IDS["class"],
                                  0, S, H, D, S, 0, 1, C, ctypes.c_void_p(0))
        assert rc == 0
        return t

    q, k, v, do = (gen_tensor(n) for n in ("q", "k", "v", "do"))
    o = torch.empty_like(q)
    lse = torch.empty(S, H, dtype=torch.float32, device="cuda")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ctx = fpdt.FPDTContext()
    fpdt.fpdt_attn_fwd(ctx, q, k, v, o, lse, S, H, H, D, 1, C, 1, fpdt.FPDT_BF16, 1)
    fpdt.fpdt_attn_bwd(ctx, o, do, dq, dk, dv, S, H, H, D, 1, C, 1, fpdt.FPDT_BF16, 1)
    torch.cuda.synchronize()
    ctx.close()
    got = {n: t[:, HEAD].float().cpu().numpy() for n, t in (("o", o), ("lse", lse), ("dq", dq), ("dk", dk),
                                                            ("dv", dv))}
    k_dev = k[:, HEAD].float().cpu().numpy()
    del q, k, v, do, o, lse, dq, dk, dv
    torch.cuda.empty_cache()

    # oracle side: the numpy twin of the generator, one head, and the closed form
    toks = np.arange(S)
    q1, k1, v1, do1 = (gen.generate(n, "class", 0, toks, H, D, S, heads=[HEAD]) for n in ("q", "k", "v", "do"))
    assert np.array_equal(k1[:, 0], k_dev)  # the device twin generated the same keys
    cls = gen.class_of(toks, S)
    kc = np.stack([k1[np.argmax(cls == c)] for c in range(int(cls.max()) + 1)])   # [K, 1, D]
    assert np.array_equal(kc[cls], k1)  # the keys are exactly the class vectors
    ro, rlse = closed_forms.class_keys_forward(q1, kc, cls, v1)
    rdq, rdk, rdv = closed_forms.class_keys_backward(q1, kc, cls, v1, do1, block=1024)
    ref = {"o": ro[:, 0], "lse": rlse[:, 0], "dq": rdq[:, 0], "dk": rdk[:, 0], "dv": rdv[:, 0]}
    errs = {n: rel_err(got[n], ref[n]) for n in ref}
    print(f"class keys, S={S}, head {HEAD}: normwise max rel err {errs}")
    assert all(e <= TOL["bf16"] for e in errs.values()), errs
