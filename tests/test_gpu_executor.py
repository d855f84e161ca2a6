"""The C++ clip-parallel executor (vinf_engine_forward_dist / _denoise_dist over a
vinf_comm) on one B200: N workers as host threads over the in-process communicator (the
shape of the reference's run_inproc_workers, transport_inproc.cpp:148-189), against the
Python stage loop (LocalGroup) that the rest of the suite pins to the oracle and the
reference. Same kernels, same exchanged bytes, same worker-order GroupNorm sums, so the
two executors must agree BITWISE; plus the oracle itself at the tolerance."""
import ctypes as C

import numpy as np
import pytest
import torch

from helpers import TOL_BF16, TOL_F32, normwise, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def en(lib):
    from paper_2406_16260_b200 import engine
    return engine


def build(en, x, n, dtype, uneven=False, n_local=8, n_global=8, groups=8, blocks=1, ablate=None):
    F, H, W, Ch = x.shape
    xd = torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)
    engines = []
    for w in range(n):
        d = en.make_desc(F, n, w, H, W, Ch, 3, groups, 1, n_local, n_global, 10.0, 800.0, 1e-5, 0.0, blocks,
                         dtype, uneven=uneven)
        e = en.ClipEngine(en.Layout(d))
        e.init_weights(1)
        e.set_ablation(ablate)
        e.x.copy_(xd[e.layout.start:e.layout.start + e.layout.f_clip])
        engines.append(e)
    return engines


def native(en, engines, use_graph=True):
    from paper_2406_16260_b200.comm import local_comms
    return en.CommGroup(local_comms(len(engines)), use_graph=use_graph)


def out(engines, attr="y"):
    torch.cuda.synchronize()
    return torch.cat([getattr(e, attr) for e in engines]).float().cpu()


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("n", [2, 3, 4])
def test_native_executor_equals_stage_loop(en, oracle, dtype, n):
    F, H, W, Ch = 48, 4, 8, 64
    x = oracle.tensor_from_seed((F, H, W, Ch), 3)
    a = build(en, x, n, dtype)
    en.forward(900.0, a, en.LocalGroup())
    b = build(en, x, n, dtype)
    en.forward(900.0, b, native(en, b))
    assert torch.equal(out(a), out(b))
    bp = oracle.build_block(Ch, 3, weight_seed=1)
    want = oracle.block_forward(x, bp, 900.0, 8, n_local=8, n_global=8)
    tol = TOL_F32 if dtype == torch.float32 else TOL_BF16
    assert normwise(out(b).numpy(), want) <= tol


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("n,Ch", [(2, 640), (4, 320)])
def test_native_executor_worker_tiles(en, oracle, dtype, n, Ch):
    # 24 frames per worker at VideoCrafter2 channel counts: the copy-warp TMA instances with
    # the O projection absorbed (bf16) under the C++ executor and graph replay, bitwise equal
    # to the stage loop and within the bar of the oracle
    F, H, W = 24 * n, 2, 4
    x = oracle.tensor_from_seed((F, H, W, Ch), 4)
    a = build(en, x, n, dtype, n_local=16, n_global=16, groups=32)
    en.forward(900.0, a, en.LocalGroup())
    b = build(en, x, n, dtype, n_local=16, n_global=16, groups=32)
    g = native(en, b)
    en.forward(900.0, b, g)
    en.forward(900.0, b, g)  # second call replays the captured graph
    assert torch.equal(out(a), out(b))
    bp = oracle.build_block(Ch, 3, weight_seed=1)
    want = oracle.block_forward(x, bp, 900.0, 32)
    tol = TOL_F32 if dtype == torch.float32 else TOL_BF16
    assert normwise(out(b).numpy(), want) <= tol


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_native_executor_uneven_two_blocks(en, dtype):
    from oracle.oracle import Oracle
    x = Oracle().tensor_from_seed((50, 2, 8, 64), 4)
    a = build(en, x, 4, dtype, uneven=True, blocks=2)
    en.forward(700.0, a, en.LocalGroup())
    b = build(en, x, 4, dtype, uneven=True, blocks=2)
    en.forward(700.0, b, native(en, b))
    assert torch.equal(out(a), out(b))


@pytest.mark.parametrize("ablate", ["conv", "groupnorm", "attention"])
def test_native_executor_ablation(en, oracle, ablate):
    x = oracle.tensor_from_seed((48, 2, 4, 64), 5)
    a = build(en, x, 3, torch.float32, ablate=ablate)
    en.forward(900.0, a, en.LocalGroup(), ablate=ablate)
    b = build(en, x, 3, torch.float32, ablate=ablate)
    en.forward(900.0, b, native(en, b))
    assert torch.equal(out(a), out(b))


def test_native_denoise_equals_stage_loop(en, oracle):
    x = oracle.tensor_from_seed((48, 2, 4, 64), 6)
    a = build(en, x, 2, torch.float32)
    en.denoise(3, a, en.LocalGroup())
    b = build(en, x, 2, torch.float32)
    en.denoise(3, b, native(en, b))
    assert torch.equal(out(a, "x"), out(b, "x"))


def test_native_executor_traffic_and_repeat(en, oracle):
    # every forward moves exactly the plan's bytes; repeated calls are bitwise stable
    x = oracle.tensor_from_seed((48, 2, 4, 64), 7)
    b = build(en, x, 3, torch.bfloat16)
    g = native(en, b)
    en.forward(900.0, b, g)
    first = out(b)
    for _ in range(2):
        en.forward(900.0, b, g)
    assert torch.equal(out(b), first)
    for e in b:
        sent = sum(xf.bytes for st in (0, 1) for xf in e.layout.exchange(st) if xf.send)
        info = g.comms[e.layout.desc.worker].info()
        assert info["bytes_sent"] == 3 * sent


def test_native_executor_profiles_sync_kinds(en, oracle):
    x = oracle.tensor_from_seed((48, 2, 4, 64), 8)
    b = build(en, x, 2, torch.bfloat16)
    for e in b:
        e.profile(True)
    en.forward(900.0, b, native(en, b))
    torch.cuda.synchronize()
    for e in b:
        names = set(e.kernel_stats())
        assert {"xchg_conv", "allreduce_gn", "xchg_attn", "conv_gemm", "attn_core"} <= names
        e.profile(False)


def test_native_executor_rejects_wrong_comm(en, oracle):
    from paper_2406_16260_b200 import _lib
    from paper_2406_16260_b200.comm import local_comms
    x = oracle.tensor_from_seed((48, 2, 4, 64), 9)
    b = build(en, x, 2, torch.bfloat16)
    comms = local_comms(2)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    with pytest.raises(_lib.ConfigError):
        _lib.check(_lib.load().vinf_engine_forward_dist(b[0]._h, C.c_double(900.0), comms[1].handle, 0, s))


def test_nccl_single_rank_graph_equals_single_worker(en, oracle):
    # NCCL communicator of one rank: the captured-graph executor path vs vinf_engine_forward
    from paper_2406_16260_b200 import _lib
    from paper_2406_16260_b200.comm import Comm
    ident = (C.c_uint8 * 128)()
    _lib.check(_lib.load().vinf_comm_nccl_unique_id(ident))
    h = C.c_void_p()
    _lib.check(_lib.load().vinf_comm_create_nccl(ident, 1, 0, C.byref(h)))
    comm = Comm(h)
    x = oracle.tensor_from_seed((24, 4, 8, 64), 10)
    a = build(en, x, 1, torch.bfloat16)
    en.forward(900.0, a)
    b = build(en, x, 1, torch.bfloat16)
    g = en.CommGroup([comm])
    for _ in range(3):  # eager, capture, replay
        en.forward(900.0, b, g)
        assert torch.equal(out(a), out(b))
