"""The N>1 host path on CPU: two / three processes over torch.distributed (gloo) run the
SAME transport code the B200 ranks run over NCCL — the reference-API sync_contexts and
group-norm all-reduce, the clip engine's workspace exchange plan (DistGroup), and the C++
executor's exchange runner (vinf_layout_run_exchange over a callback communicator: the
code path vinf_engine_forward_dist takes, with gloo in place of NCCL)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, errq):
    try:
        sys.path.insert(0, ROOT)
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        from paper_2406_16260_b200 import _lib
        from paper_2406_16260_b200 import clip_parallel as cp
        from paper_2406_16260_b200 import engine as en
        from paper_2406_16260_b200.transport import DistTransport

        t = DistTransport()
        # (1) reference-API sync: halo + global frames land bitwise (test_clip_parallel.cpp:94-149)
        F = 48
        full = torch.arange(F * 2 * 2 * 4, dtype=torch.float32).reshape(F, 2, 2, 4)
        plan = cp.make_plan(F, world)
        clip = full[rank * plan.f_clip:(rank + 1) * plan.f_clip].contiguous()
        ctx = cp.sync_contexts(t, plan, cp.LayerHaloSpec(cp.LayerKind.Attention, 2, 8), clip)
        fc = plan.f_clip
        if rank > 0:
            assert torch.equal(ctx.c_pre, full[rank * fc - 2:rank * fc])
        else:
            assert ctx.c_pre is None
        if rank + 1 < world:
            assert torch.equal(ctx.c_post, full[(rank + 1) * fc:(rank + 1) * fc + 2])
        else:
            assert ctx.c_post is None
        idx = cp.build_global_index_set(F, 8)
        assert torch.equal(ctx.c_global, full[idx])
        # measured bytes vs the reference's closed form is not expected to match exactly:
        # globals go point-to-point to each peer rather than around a ring; the closed form
        # is the reference's ring and is reported separately.
        # (2) all-reduce of f64 partial sums
        s = torch.full((4,), float(rank + 1), dtype=torch.float64)
        t.allreduce_sum_(s)
        assert torch.allclose(s, torch.full((4,), float(world * (world + 1) / 2), dtype=torch.float64))
        # (3) engine exchange plan over the transport, on a CPU workspace
        n_local, n_global, Fe = 8, 16, 48
        L = en.Layout(en.make_desc(Fe, world, rank, 2, 2, 16, groups=4, n_local=n_local,
                                   n_global=n_global, dtype=torch.bfloat16))

        class FakeEngine:  # the exchange only needs the layout and the workspace
            pass

        e = FakeEngine()
        e.layout = L
        e.ws = torch.zeros(L.workspace_bytes, dtype=torch.uint8)
        off, _, fb = L.region(_lib.VINF_BUF_ATTN_IN)
        ha, fc = n_local // 2, Fe // world
        for f in range(fc):
            e.ws[off + (ha + f) * fb: off + (ha + f + 1) * fb] = rank * fc + f
        en.DistGroup(t).exchange([e], _lib.VINF_XCHG_ATTN)
        fr = lambda k: e.ws[off + k * fb: off + (k + 1) * fb]  # noqa: E731
        if rank > 0:
            for k in range(ha):
                assert (fr(k) == rank * fc - ha + k).all()
        if rank + 1 < world:
            for k in range(ha):
                assert (fr(ha + fc + k) == (rank + 1) * fc + k).all()
        lo = rank * fc - (ha if rank > 0 else 0)
        hi = (rank + 1) * fc + (ha if rank + 1 < world else 0)
        remote = [g for g in cp.build_global_index_set(Fe, n_global) if not lo <= g < hi]
        for slot, g in enumerate(remote):
            assert (fr(2 * ha + fc + slot) == g).all()
        # (4) the C++ executor: the same plans through vinf_layout_run_exchange over an
        # OpsComm (gloo on host pointers), both stages, plus its f64 all-reduce
        from paper_2406_16260_b200.comm import GlooPointerTransport, OpsComm
        comm = OpsComm(GlooPointerTransport())
        ws = torch.zeros(L.workspace_bytes, dtype=torch.uint8)
        coff, _, cfb = L.region(_lib.VINF_BUF_CONV_IN)
        for f in range(fc):
            ws[off + (ha + f) * fb: off + (ha + f + 1) * fb] = (rank * fc + f) % 251
            ws[coff + (1 + f) * cfb: coff + (2 + f) * cfb] = (rank * fc + f + 7) % 251
        base = ws.data_ptr()
        for stage in (_lib.VINF_XCHG_CONV, _lib.VINF_XCHG_ATTN):
            _lib.check(_lib.load().vinf_layout_run_exchange(L._h, stage, base, comm.handle, None))
        assert not comm.errors, comm.errors
        fa = lambda k: ws[off + k * fb: off + (k + 1) * fb]  # noqa: E731
        fcv = lambda k: ws[coff + k * cfb: coff + (k + 1) * cfb]  # noqa: E731
        if rank > 0:
            assert (fcv(0) == (rank * fc - 1 + 7) % 251).all()
            for k in range(ha):
                assert (fa(k) == (rank * fc - ha + k) % 251).all()
        else:
            assert (fcv(0) == 0).all()
        if rank + 1 < world:
            assert (fcv(1 + fc) == ((rank + 1) * fc + 7) % 251).all()
            for k in range(ha):
                assert (fa(ha + fc + k) == ((rank + 1) * fc + k) % 251).all()
        for slot, g in enumerate(remote):
            assert (fa(2 * ha + fc + slot) == g % 251).all()
        info = comm.info()
        sent = sum(x.bytes for st in (0, 1) for x in L.exchange(st) if x.send)
        assert info["bytes_sent"] == sent and info["rank"] == rank and info["nranks"] == world
        red = torch.arange(6, dtype=torch.float64) * (rank + 1)
        comm.allreduce_sum_f64(red.data_ptr(), 6)
        assert torch.equal(red, torch.arange(6, dtype=torch.float64) * (world * (world + 1) / 2))
        # a mismatched communicator is refused before any message moves
        with pytest.raises(_lib.ConfigError):
            L0 = en.Layout(en.make_desc(Fe, world, (rank + 1) % world, 2, 2, 16, groups=4, n_local=n_local,
                                        n_global=n_global, dtype=torch.bfloat16))
            _lib.check(_lib.load().vinf_layout_run_exchange(L0._h, 0, base, comm.handle, None))
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as ex:  # noqa: BLE001
        import traceback
        errq.put(f"rank {rank}: {traceback.format_exc()}")
        raise


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_world(world, lib):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs)
