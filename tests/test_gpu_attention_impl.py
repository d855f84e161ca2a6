"""Both feeds of the attention core (the TMA ring and the cp.async ring, attention_core.cu /
attention_cpasync.cu) on the same inputs, each forced through vinf_debug_attention_impl, against
the oracle (attend_tokens, ops.cpp:209-241): narrow and wide K/V tiles, multi-head, both
arithmetic modes. launch_attention_core picks one by configuration; this checks the other one
too, so neither is an untested path."""
import numpy as np
import pytest
import torch

from helpers import TOL_BF16, TOL_F32, normwise, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture
def impl(lib):
    from paper_2406_16260_b200 import _lib
    old = _lib.load().vinf_debug_attention_impl(0)
    yield lambda k: _lib.load().vinf_debug_attention_impl(k)
    _lib.load().vinf_debug_attention_impl(old)


CASES = [  # F, H, W, C, heads, n_local, n_global
    (24, 4, 8, 128, 1, 16, 16),   # narrow (24 K/V frames)
    (96, 2, 4, 128, 2, 32, 64),   # wide: band + many globals
    (24, 2, 8, 320, 8, 16, 16),   # d = 40 (chunk zero-filled past the head dim)
    (24, 4, 8, 640, 1, 16, 16),   # the 24-frame clip at C = 640 (the copy-warp instance)
    (24, 3, 5, 320, 1, 8, 4),     # 15 positions (a partial 4-position item), sparse globals
]



@pytest.mark.parametrize("which", [1, 2])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("case", CASES)
def test_attention_feed_vs_oracle(impl, oracle, which, dtype, case):
    from paper_2406_16260_b200 import engine as en
    F, H, W, C, heads, nl, ng = case
    impl(which)
    x = oracle.tensor_from_seed((F, H, W, C), 11)
    d = en.make_desc(F, 1, 0, H, W, C, 3, 8, heads, nl, ng, 10.0, 800.0, 1e-5, 0.0, 1, dtype)
    e = en.ClipEngine(en.Layout(d))
    e.init_weights(1)
    e.x.copy_(torch.from_numpy(x).to("cuda", dtype))
    en.forward(900.0, [e])
    got = to_np(e.y)
    bp = oracle.build_block(C, 3, weight_seed=1)
    scale = float(np.float32(1) / np.sqrt(np.float32(C // heads)))
    want = oracle.block_forward(x, bp, 900.0, 8, n_local=nl, n_global=ng, heads=heads, scale=scale)
    tol = TOL_F32 if dtype == torch.float32 else TOL_BF16
    assert np.isfinite(got).all()
    assert normwise(got, want) <= tol
