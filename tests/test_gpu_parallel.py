"""GPU parity of the distributed forms (clip_parallel.cpp:194-341) and the clip engine:
N workers run as threads (LocalTransport) or as N engines on one GPU (LocalGroup),
exactly the reference's in-process multi-worker test strategy."""
import numpy as np
import pytest
import torch

from helpers import TOL_BF16, TOL_F32, normwise, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods(lib):
    from paper_2406_16260_b200 import clip_parallel, engine, ops, transport
    return ops, clip_parallel, engine, transport


def dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda").to(dtype)


# ---- reference-API distributed forms ---------------------------------------------


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_conv_parallel_equals_oracle_form(mods, oracle, n):
    # test_clip_parallel.cpp:151-170: distributed conv == sequential conv, bitwise
    ops, cp, _, tr = mods
    x = dev(oracle.tensor_from_seed((16, 2, 4, 32), 41))
    bp = oracle.build_block(32, 5, weight_seed=42)
    k = ops.ConvKernel(5, dev(bp.conv_w), dev(bp.conv_b))
    want = ops.temporal_conv(x, k)
    plan = cp.make_plan(16, n)
    clips = cp.partition(x, n)
    spec = cp.LayerHaloSpec(cp.LayerKind.Conv, k.halo(), 0)

    def body(t):
        ctx = cp.sync_contexts(t, plan, spec, clips[t.rank])
        return cp.conv_parallel(plan, t.rank, clips[t.rank], ctx, k)

    got = torch.cat(tr.run_local_workers(n, body))
    torch.cuda.synchronize()
    assert torch.equal(got, want)


@pytest.mark.parametrize("n", [1, 2, 4])
@pytest.mark.parametrize("t", [700.0, 900.0])
def test_attention_parallel_equals_oracle_form(mods, oracle, n, t):
    # test_clip_parallel.cpp:263-297: distributed attention == dual_scope_reference
    ops, cp, _, tr = mods
    F, C = 32, 32
    x = dev(oracle.tensor_from_seed((F, 2, 2, C), 51))
    bp = oracle.build_block(C, weight_seed=52)
    p = ops.AttentionParams(C, dev(bp.wq), dev(bp.wk), dev(bp.wv), dev(bp.wo))
    cfg = ops.DualScopeConfig(8, 6, 10.0, 800.0)
    want = ops.dual_scope_reference(x, t, p, cfg)
    plan = cp.make_plan(F, n)
    clips = cp.partition(x, n)
    spec = cp.LayerHaloSpec(cp.LayerKind.Attention, cfg.n_local // 2, cfg.n_global)

    def body(tp):
        ctx = cp.sync_contexts(tp, plan, spec, clips[tp.rank])
        return cp.attention_parallel(plan, tp.rank, clips[tp.rank], ctx, t, p, cfg)

    got = torch.cat(tr.run_local_workers(n, body))
    torch.cuda.synchronize()
    # the distributed form keeps the global frames as separate K/V rows (the reference's
    # [ext | globals] row table, clip_parallel.cpp:277-280) where the sequential form
    # shares a column between a window frame and the same global frame, so P is split into
    # bf16 hi/lo planes over different column sums: equal to the bf16x3 precision (~2^-16)
    assert normwise(to_np(got), to_np(want)) <= 2e-5
    # and against the CPU oracle's own distributed form on worker 1
    if n > 1:
        xs = oracle.tensor_from_seed((F, 2, 2, C), 51)
        fc = F // n
        h = cfg.n_local // 2
        gidx = oracle.build_global_index_set(F, cfg.n_global)
        sc = float(np.float32(1) / np.sqrt(np.float32(C)))
        w1 = oracle.attention_parallel(F, n, 1, xs[fc:2 * fc], xs[fc - h:fc],
                                       xs[2 * fc:2 * fc + h] if n > 2 else None, xs[gidx], t,
                                       bp.wq, bp.wk, bp.wv, bp.wo, sc, cfg.n_local, cfg.n_global,
                                       10.0, 800.0)
        assert normwise(to_np(got[fc:2 * fc]), w1) <= TOL_F32


@pytest.mark.parametrize("n", [1, 2, 4])
def test_group_norm_parallel(mods, oracle, n):
    ops, cp, _, tr = mods
    x = dev(oracle.tensor_from_seed((16, 2, 4, 32), 61) * 2.0 + 0.25)
    bp = oracle.build_block(32)
    p = ops.GroupNormParams(4, dev(bp.gamma), dev(bp.beta))
    want = ops.group_norm(x, p)
    plan = cp.make_plan(16, n)
    clips = cp.partition(x, n)
    got = torch.cat(tr.run_local_workers(
        n, lambda t: cp.group_norm_parallel(t, plan, clips[t.rank].contiguous(), p)))
    assert normwise(to_np(got), to_np(want)) <= 1e-6


def test_group_norm_footnote_case(mods):
    # test_clip_parallel.cpp:224-261: clips {0,0} and {2,2} -> global sigma = 1, not 0
    ops, cp, _, tr = mods
    C = 8
    clips = [torch.zeros((2, 1, 1, C), device="cuda"), torch.full((2, 1, 1, C), 2.0, device="cuda")]
    p = ops.GroupNormParams(1, torch.ones(C, device="cuda"), torch.zeros(C, device="cuda"))
    plan = cp.make_plan(4, 2)
    out = tr.run_local_workers(2, lambda t: cp.group_norm_parallel(t, plan, clips[t.rank], p))
    want = -1.0 / np.sqrt(1.0 + 1e-5)
    assert np.allclose(to_np(out[0]), want, atol=1e-6) and np.allclose(to_np(out[1]), -want, atol=1e-6)


def test_context_size_mismatch_is_protocol_error(mods, oracle):
    ops, cp, _, _ = mods
    bp = oracle.build_block(16)
    k = ops.ConvKernel(3, dev(bp.conv_w), dev(bp.conv_b))
    plan = cp.make_plan(8, 2)
    v = torch.zeros((4, 1, 1, 16), device="cuda")
    with pytest.raises(ops.ProtocolError):
        cp.conv_parallel(plan, 1, v, cp.TemporalContext(), k)  # worker 1 needs c_pre


# ---- clip engine -----------------------------------------------------------------


def _engine(mods, dtype, **kw):
    _, _, en, _ = mods
    L = en.Layout(en.make_desc(dtype=dtype, **kw))
    e = en.ClipEngine(L)
    return e


BLOCK = dict(frames=24, height=4, width=8, channels=64, groups=8, n_local=16, n_global=16)


@pytest.mark.parametrize("dtype,tol", [(torch.float32, TOL_F32), (torch.bfloat16, TOL_BF16)])
@pytest.mark.parametrize("t", [700.0, 900.0])
def test_engine_single_worker_vs_oracle(mods, oracle, dtype, tol, t):
    _, _, en, _ = mods
    e = _engine(mods, dtype, **BLOCK)
    e.init_weights(1)
    x = oracle.tensor_from_seed((24, 4, 8, 64), 0)
    e.x.copy_(dev(x, dtype))
    en.forward(t, [e])
    bp = oracle.build_block(64, 3, weight_seed=1)
    want = oracle.block_forward(x if dtype == torch.float32 else to_np(dev(x, dtype)), bp, t, 8)
    got = to_np(e.y)
    assert normwise(got, want) <= tol, normwise(got, want)


@pytest.mark.parametrize("C", [320, 640])
def test_engine_production_channels(mods, oracle, C):
    # the bench's channel counts (VideoCrafter2 levels) through the whole fused block,
    # both modes, vs the CPU oracle; and the bf16 engine is bitwise reproducible
    _, _, en, _ = mods
    kw = dict(frames=24, height=2, width=4, channels=C, groups=32, n_local=16, n_global=16)
    x = oracle.tensor_from_seed((24, 2, 4, C), 0)
    bp = oracle.build_block(C, 3, weight_seed=1)
    for dtype, tol in ((torch.float32, TOL_F32), (torch.bfloat16, TOL_BF16)):
        e = _engine(mods, dtype, **kw)
        e.init_weights(1)
        xd = dev(x, dtype)
        e.x.copy_(xd)
        en.forward(900.0, [e])
        y1 = e.y.clone()
        want = oracle.block_forward(to_np(xd), bp, 900.0, 32)
        assert normwise(to_np(y1), want) <= tol, (dtype, normwise(to_np(y1), want))
        e.x.copy_(xd)
        en.forward(900.0, [e])
        torch.cuda.synchronize()
        assert torch.equal(e.y, y1)


@pytest.mark.parametrize("H,W,C,groups", [(40, 41, 64, 8), (12, 23, 640, 32)])
def test_engine_many_tiles_per_cta(mods, oracle, H, W, C, groups):
    # enough rows that persistent GEMM CTAs run several tiles (the TMA residual ring crosses
    # tile boundaries, the quadrant warps swap chunk parity on odd tiles, the conv's column
    # statistics accumulate per CTA), with a partial last row tile and, at C = 640, a
    # partial last column tile (N tile 224); bf16 engine vs the CPU oracle, and repeatable
    _, _, en, _ = mods
    F = 24
    kw = dict(frames=F, height=H, width=W, channels=C, groups=groups, n_local=16, n_global=16)
    x = oracle.tensor_from_seed((F, H, W, C), 4)
    bp = oracle.build_block(C, 3, weight_seed=1)
    e = _engine(mods, torch.bfloat16, **kw)
    e.init_weights(1)
    xd = dev(x, torch.bfloat16)
    e.x.copy_(xd)
    en.forward(700.0, [e])
    y1 = e.y.clone()
    want = oracle.block_forward(to_np(xd), bp, 700.0, groups)
    assert normwise(to_np(y1), want) <= TOL_BF16, normwise(to_np(y1), want)
    e.x.copy_(xd)
    en.forward(700.0, [e])
    torch.cuda.synchronize()
    assert torch.equal(e.y, y1)


def test_engine_set_block_equals_init_weights(mods, oracle):
    _, _, en, _ = mods
    bp = oracle.build_block(64, 3, weight_seed=5)
    e1 = _engine(mods, torch.float32, **BLOCK)
    e1.init_weights(5)
    e2 = _engine(mods, torch.float32, **BLOCK)
    e2.set_block(0, *[dev(a) for a in bp.arrays()])
    x = dev(oracle.tensor_from_seed((24, 4, 8, 64), 3))
    for e in (e1, e2):
        e.x.copy_(x)
        en.forward(900.0, [e])
    torch.cuda.synchronize()
    assert torch.equal(e1.y, e2.y)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_engine_is_deterministic(mods, oracle, dtype):
    # no atomics on the value path: repeated runs (and two engines) agree bitwise
    _, _, en, _ = mods
    x = dev(oracle.tensor_from_seed((24, 4, 8, 64), 8), dtype)
    outs = []
    for _ in range(2):
        e = _engine(mods, dtype, **BLOCK)
        e.init_weights(2)
        for _ in range(2):
            e.x.copy_(x)
            en.forward(900.0, [e])
            outs.append(e.y.clone())
    torch.cuda.synchronize()
    assert all(torch.equal(o, outs[0]) for o in outs[1:])


@pytest.mark.parametrize("n", [2, 3, 4, 6])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_engine_clip_parallel_equals_single(mods, oracle, n, dtype):
    _, _, en, _ = mods
    F = 48
    kw = dict(BLOCK, frames=F)
    x = dev(oracle.tensor_from_seed((F, 4, 8, 64), 7), dtype)
    single = _engine(mods, dtype, **kw)
    single.init_weights(1)
    single.x.copy_(x)
    en.forward(900.0, [single])
    engines = []
    fc = F // n
    for w in range(n):
        e = _engine(mods, dtype, workers=n, worker=w, **kw)
        e.init_weights(1)
        e.x.copy_(x[w * fc:(w + 1) * fc])
        engines.append(e)
    en.forward(900.0, engines)
    got = torch.cat([e.y for e in engines])
    torch.cuda.synchronize()
    # identical arithmetic except the summation grouping of the GN statistics and of the
    # softmax normaliser (columns follow each worker's K/V list); in bf16 that can move an
    # output by one unit in the last place (2^-8 relative)
    bound = 1e-5 if dtype == torch.float32 else 2.0 ** -8
    assert normwise(to_np(got), to_np(single.y)) <= bound
    if dtype == torch.float32:
        bp = oracle.build_block(64, 3, weight_seed=1)
        want = oracle.block_forward(to_np(x), bp, 900.0, 8)
        assert normwise(to_np(got), want) <= TOL_F32


def test_engine_two_blocks(mods, oracle):
    _, _, en, _ = mods
    e = _engine(mods, torch.float32, blocks=2, **BLOCK)
    e.init_weights(9)
    x = oracle.tensor_from_seed((24, 4, 8, 64), 4)
    e.x.copy_(dev(x))
    en.forward(900.0, [e])
    b0 = oracle.build_block(64, 3, weight_seed=9, block=0)
    b1 = oracle.build_block(64, 3, weight_seed=9, block=1)
    want = oracle.block_forward(oracle.block_forward(x, b0, 900.0, 8), b1, 900.0, 8)
    assert normwise(to_np(e.y), want) <= TOL_F32


@pytest.mark.parametrize("blocks,steps,n", [(1, 4, 1), (2, 3, 1), (1, 3, 2), (2, 2, 4)])
def test_denoise_matches_reference_execute_run(mods, reference, blocks, steps, n):
    # The reference's whole public run path (execute_run -> worker_denoise, runner.cpp:26-73,
    # pipeline.cpp:174-191): `steps` Euler steps of a `blocks`-block stack, from the seeded
    # latent, sequential (reference) vs clip-parallel over n engines (here).
    _, _, en, _ = mods
    F, H, W, Cc = 16, 4, 4, 32
    wall, x0 = reference.execute_run(F, H, W, Cc, groups=4, n_local=8, n_global=4, blocks=blocks,
                                     steps=steps, want_x0=True)
    from paper_2406_16260_b200 import ops
    x = ops.tensor_from_seed((F, H, W, Cc), 0)
    engines = []
    fc = F // n
    for w in range(n):
        e = _engine(mods, torch.float32, frames=F, workers=n, worker=w, height=H, width=W,
                    channels=Cc, groups=4, n_local=8, n_global=4, blocks=blocks)
        e.init_weights(1)
        e.x.copy_(x[w * fc:(w + 1) * fc])
        engines.append(e)
    en.denoise(steps, engines)
    got = torch.cat([e.x for e in engines])
    assert normwise(to_np(got), x0) <= TOL_F32, normwise(to_np(got), x0)


def test_engine_matches_reference_run_path(mods, reference):
    # The reference's own public run path, one Euler step of one block (runner.cpp:26-41):
    # x0 = x - (1/steps) * eps_theta(x, t=1000)
    _, _, en, _ = mods
    F, H, W, Cc = 16, 4, 4, 32
    wall, x0 = reference.execute_run(F, H, W, Cc, groups=4, n_local=8, n_global=4, steps=1,
                                     want_x0=True)
    e = _engine(mods, torch.float32, frames=F, height=H, width=W, channels=Cc, groups=4,
                n_local=8, n_global=4)
    e.init_weights(1)
    from paper_2406_16260_b200 import ops
    x = ops.tensor_from_seed((F, H, W, Cc), 0)
    e.x.copy_(x)
    en.forward(1000.0, [e])
    got = to_np(x) - to_np(e.y)
    assert normwise(got, x0) <= TOL_F32


@pytest.mark.parametrize("n", [1, 3])
def test_gn_fold_matches_apply_path(mods, oracle, n, monkeypatch):
    # bf16 mode folds GroupNorm into W_qkv (W diag(s), bias W t) and the O GEMM residual;
    # VINF_NO_GN_FOLD=1 keeps the explicit apply kernel. Both are bf16 evaluations of the
    # same block: they agree to bf16 rounding, and each meets the oracle tolerance.
    _, _, en, _ = mods
    F = 24
    kw = dict(BLOCK, frames=F)
    x = dev(oracle.tensor_from_seed((F, 4, 8, 64), 11), torch.bfloat16)
    outs = {}
    for fold in (True, False):
        if fold:
            monkeypatch.delenv("VINF_NO_GN_FOLD", raising=False)
        else:
            monkeypatch.setenv("VINF_NO_GN_FOLD", "1")
        engines = []
        for w in range(n):
            e = _engine(mods, torch.bfloat16, workers=n, worker=w, **kw)
            e.init_weights(3)
            e.x.copy_(x[w * F // n:(w + 1) * F // n])
            engines.append(e)
        for t in (900.0, 700.0):
            en.forward(t, engines)
            outs[(fold, t)] = torch.cat([e.y for e in engines]).clone()
    bp = oracle.build_block(64, 3, weight_seed=3)
    for t in (900.0, 700.0):
        want = oracle.block_forward(to_np(x), bp, t, 8)
        a, b = to_np(outs[(True, t)]), to_np(outs[(False, t)])
        assert normwise(a, b) <= 1e-2, normwise(a, b)
        assert normwise(a, want) <= TOL_BF16 and normwise(b, want) <= TOL_BF16
