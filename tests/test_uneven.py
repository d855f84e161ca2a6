"""Uneven clips (extension; the reference requires workers | frames, clip_parallel.cpp:56-59):
worker w owns frames [floor(w*F/N), floor((w+1)*F/N)), e.g. 2,300 frames over 8 GPUs.
The layout/exchange plan is checked on CPU; on the GPU the clip-parallel engines must
reproduce the single-worker result."""
import numpy as np
import pytest
import torch

from helpers import TOL_F32, dev, normwise, to_np


def _layouts(F, N, **kw):
    from paper_2406_16260_b200 import engine as en
    return [en.Layout(en.make_desc(F, N, w, uneven=True, **kw)) for w in range(N)]


@pytest.mark.parametrize("F,N", [(19, 4), (2300, 8), (16, 3), (24, 5)])
def test_uneven_partition_and_exchange_plan(lib, F, N):
    kw = dict(height=2, width=2, channels=8, groups=2, n_local=4, n_global=min(16, F))
    Ls = _layouts(F, N, **kw)
    starts = [L.start for L in Ls]
    sizes = [L.f_clip for L in Ls]
    assert starts == [w * F // N for w in range(N)]
    assert sum(sizes) == F and max(sizes) - min(sizes) <= 1
    for stage in (0, 1):
        xs = [L.exchange(stage) for L in Ls]
        for w in range(N):
            for x in xs[w]:
                if x.send:
                    continue
                src = [s for s in xs[x.peer] if s.send and s.peer == w and s.tag == x.tag]
                assert len(src) == 1 and src[0].bytes == x.bytes, (stage, w, x.tag)
    # every global frame outside a worker's synchronised window arrives exactly once
    from paper_2406_16260_b200 import ops
    gset = ops.build_global_index_set(F, kw["n_global"])
    ha = kw["n_local"] // 2
    for w, L in enumerate(Ls):
        lo = starts[w] - (ha if w > 0 else 0)
        hi = starts[w] + sizes[w] + (ha if w + 1 < N else 0)
        remote = [g for g in gset if not lo <= g < hi]
        recv = [x for x in L.exchange(1) if not x.send and x.tag >= 3000 and x.tag % 4 == 0]  # plane 0
        assert len(recv) == len(remote)


def test_even_split_still_required_without_flag(lib):
    from paper_2406_16260_b200 import _lib, engine as en
    with pytest.raises(_lib.ConfigError):
        en.Layout(en.make_desc(19, 4, 0, height=2, width=2, channels=8, groups=2, n_local=4, n_global=4))
    with pytest.raises(_lib.ConfigError):  # the halo must fit the smallest clip
        en.Layout(en.make_desc(10, 4, 0, height=2, width=2, channels=8, groups=2, n_local=6,
                               n_global=4, uneven=True))


@pytest.mark.gpu
@pytest.mark.parametrize("F,N,blocks,dtype", [(19, 4, 1, torch.float32), (16, 3, 2, torch.float32),
                                              (19, 4, 2, torch.bfloat16)])
def test_uneven_engines_match_single_worker(lib, F, N, blocks, dtype):
    # bf16 runs the GroupNorm-folded projections: raw frames cross the uneven clip edges
    from paper_2406_16260_b200 import engine as en, ops
    kw = dict(height=4, width=4, channels=32, groups=4, n_local=4, n_global=5, blocks=blocks,
              dtype=dtype)
    x = ops.tensor_from_seed((F, 4, 4, 32), 0)
    one = en.ClipEngine(en.Layout(en.make_desc(F, 1, 0, **kw)))
    one.init_weights(1)
    one.x.copy_(dev(x, dtype))
    en.denoise(2, [one])
    engines = []
    for w in range(N):
        e = en.ClipEngine(en.Layout(en.make_desc(F, N, w, uneven=True, **kw)))
        e.init_weights(1)
        e.x.copy_(dev(x[e.layout.start:e.layout.start + e.layout.f_clip], dtype))
        engines.append(e)
    en.denoise(2, engines)
    got = np.concatenate([to_np(e.x) for e in engines])
    want = to_np(one.x)
    # fp32: summation grouping only; bf16: plus one rounding step per block (2^-8 each)
    bound = 1e-5 if dtype == torch.float32 else 2.0 ** -7
    assert normwise(got, want) <= bound, normwise(got, want)
