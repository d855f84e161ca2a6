"""Clip engine: the preallocated, fused temporal block stack of one worker
(eps_theta_worker, pipeline.cpp:145-172) and the stage loop that interleaves it with the
paper's 3-step context sync.

    layout = Layout(EngineDesc(...))         # pure host: buffers + exchange plan
    eng = ClipEngine(layout)                 # one device workspace, weights on device
    eng.init_weights(weight_seed=1)          # build_model (pipeline.cpp:35-67) on device
    eng.x.copy_(clip)                        # [f_clip, H, W, C] in the engine dtype
    forward(t=900.0, engines=[eng])          # single worker: one C call
    forward(t, [eng], DistGroup(transport))  # clip-parallel, Python stage loop over torch.distributed
    forward(t, [eng], CommGroup([NcclComm.create()]))  # clip-parallel, the C++ executor over NCCL

Exchanges are the workspace byte ranges the C++ layout lists (halo frames into the
neighbours' halo slots, remote global frames into global slots), so the transport moves
bf16 planes straight between the producers' and consumers' operand buffers.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import EngineDesc
from .transport import Msg, Transport

_TORCH_DT = {_lib.VINF_F32: torch.float32, _lib.VINF_BF16: torch.bfloat16}
_ABLATE = {None: _lib.VINF_ABLATE_NONE, "none": _lib.VINF_ABLATE_NONE, "conv": _lib.VINF_ABLATE_CONV,
           "groupnorm": _lib.VINF_ABLATE_GROUPNORM, "attention": _lib.VINF_ABLATE_ATTENTION}


def make_desc(frames, workers=1, worker=0, height=32, width=32, channels=320, taps=3, groups=32,
              heads=1, n_local=16, n_global=16, bias=10.0, t_star=800.0, epsilon=1e-5,
              scale=0.0, blocks=1, dtype=torch.float32, uneven=False) -> EngineDesc:
    dt = _lib.VINF_F32 if dtype == torch.float32 else _lib.VINF_BF16
    return EngineDesc(frames, workers, worker, height, width, channels, taps, groups, heads,
                      n_local, n_global, bias, t_star, epsilon, scale, blocks, dt, int(uneven))


class Layout:
    """Host-side workspace layout + exchange plan (vinf_layout_*); no CUDA needed."""

    def __init__(self, desc: EngineDesc):
        self.desc = desc
        self._lib = _lib.load()
        h = C.c_void_p()
        _lib.check(self._lib.vinf_layout_create(C.byref(desc), C.byref(h)))
        self._h = h
        n = C.c_uint64()
        _lib.check(self._lib.vinf_layout_workspace_bytes(h, C.byref(n)))
        self.workspace_bytes = n.value
        st, fc = C.c_uint32(), C.c_uint32()
        _lib.check(self._lib.vinf_layout_clip(h, C.byref(st), C.byref(fc)))
        self.start, self.f_clip = st.value, fc.value
        self.dtype = _TORCH_DT[desc.dtype]

    def region(self, which: int):
        off, n, fb = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _lib.check(self._lib.vinf_layout_region(self._h, which, C.byref(off), C.byref(n),
                                                C.byref(fb)))
        return off.value, n.value, fb.value

    def exchange(self, stage: int) -> list[_lib.Xfer]:
        """The stage's transfer list (computed once per layout; the plan is immutable)."""
        cache = self.__dict__.setdefault("_xcache", {})
        if stage not in cache:
            n = C.c_uint32()
            _lib.check(self._lib.vinf_layout_exchange(self._h, stage, None, 0, C.byref(n)))
            arr = (_lib.Xfer * max(n.value, 1))()
            _lib.check(self._lib.vinf_layout_exchange(self._h, stage, arr, n.value, C.byref(n)))
            cache[stage] = [arr[i] for i in range(n.value)]
        return cache[stage]

    def reference_traffic(self):
        a, b, c = (C.c_uint64 * 3)(), (C.c_uint64 * 3)(), (C.c_uint64 * 3)()
        _lib.check(self._lib.vinf_layout_reference_traffic(self._h, a, b, c))
        return list(a), list(b), list(c)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None and _lib._lib is not None:
            _lib._lib.vinf_layout_destroy(self._h)
            self._h = None


class ClipEngine:
    def __init__(self, layout: Layout, device=None, workspace: torch.Tensor | None = None):
        self.layout = layout
        self.device = torch.device(device or "cuda")
        self.ws = workspace if workspace is not None else torch.empty(
            layout.workspace_bytes, dtype=torch.uint8, device=self.device)
        d = layout.desc
        self.shape = (layout.f_clip, d.height, d.width, d.channels)
        h = C.c_void_p()
        _lib.check(_lib.load().vinf_engine_create(layout._h, C.c_void_p(self.ws.data_ptr()),
                                                  self._stream(), C.byref(h)))
        self._h = h
        xo, xn, _ = layout.region(_lib.VINF_BUF_X)
        self.x = self.ws[xo:xo + xn].view(layout.dtype).view(self.shape)
        yp = C.c_void_p()
        _lib.check(_lib.load().vinf_engine_io(h, None, C.byref(yp)))
        yo = yp.value - self.ws.data_ptr()
        self.y = self.ws[yo:yo + xn].view(layout.dtype).view(self.shape)
        so, sn, _ = layout.region(_lib.VINF_BUF_GN_SUMS)
        self.gn_sums = self.ws[so:so + sn].view(torch.float64).view(2, d.groups)

    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def init_weights(self, weight_seed: int = 1) -> None:
        _lib.check(_lib.load().vinf_engine_init_weights(self._h, weight_seed, self._stream()))

    def set_block(self, b: int, stub_a, stub_c, conv_w, conv_b, gamma, beta, wq, wk, wv, wo):
        ts = [t.detach().to(device=self.device, dtype=torch.float32).contiguous()
              for t in (stub_a, stub_c, conv_w, conv_b, gamma, beta, wq, wk, wv, wo)]
        _lib.check(_lib.load().vinf_engine_set_block(self._h, b, *[C.c_void_p(t.data_ptr()) for t in ts],
                                                     self._stream()))
        torch.cuda.current_stream(self.device).synchronize()

    def stage(self, block: int, stage: int, t: float) -> None:
        _lib.check(_lib.load().vinf_engine_stage(self._h, block, stage, C.c_double(t), self._stream()))

    def forward_single(self, t: float) -> None:
        _lib.check(_lib.load().vinf_engine_forward(self._h, C.c_double(t), self._stream()))

    def euler(self, lam: float) -> None:
        """x -= lam * y (euler_update_inplace, pipeline.cpp:93-100)."""
        _lib.check(_lib.load().vinf_engine_euler(self._h, C.c_double(lam), self._stream()))

    def set_ablation(self, kind: str | None) -> None:
        """Sync ablation (the reference's `ablate` key): None | "conv" | "groupnorm" |
        "attention". forward()/denoise() must be given the same kind so the group skips
        that exchange."""
        _lib.check(_lib.load().vinf_engine_set_ablation(self._h, _ABLATE[kind]))

    def denoise_single(self, steps: int) -> None:
        _lib.check(_lib.load().vinf_engine_denoise(self._h, steps, self._stream()))

    def launches(self) -> int:
        return int(_lib.load().vinf_engine_launches(self._h))

    def profile(self, enable: bool = True) -> None:
        _lib.check(_lib.load().vinf_engine_profile(self._h, int(enable)))

    def kernel_stats(self) -> dict:
        """{kernel name: (total ms, launches)} since the last read (needs profile())."""
        names = C.create_string_buffer(1024)
        ms = (C.c_double * 32)()
        cnt = (C.c_uint64 * 32)()
        n = C.c_uint32()
        _lib.check(_lib.load().vinf_engine_kernel_stats(self._h, names, 1024, ms, cnt, 32,
                                                        C.byref(n)))
        keys = names.value.decode().split(",") if n.value else []
        return {k: (ms[i], int(cnt[i])) for i, k in enumerate(keys)}

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None and _lib._lib is not None:
            _lib._lib.vinf_engine_destroy(self._h)
            self._h = None


class LocalGroup:
    """All workers' engines in this process (e.g. N clips on one GPU): exchanges are
    device-to-device copies between workspaces, all-reduces sum in worker order."""

    def exchange(self, engines: list[ClipEngine], stage: int) -> None:
        by_worker = {e.layout.desc.worker: e for e in engines}
        lists = {w: e.layout.exchange(stage) for w, e in by_worker.items()}
        for w, xs in lists.items():
            for x in xs:
                if x.send:
                    continue
                src = [s for s in lists[x.peer] if s.send and s.peer == w and s.tag == x.tag]
                if len(src) != 1 or src[0].bytes != x.bytes:
                    raise _lib.ProtocolError(f"unmatched transfer into worker {w} tag {x.tag}")
                s = src[0]
                dst_ws, src_ws = by_worker[w].ws, by_worker[x.peer].ws
                dst_ws[x.offset:x.offset + x.bytes].copy_(src_ws[s.offset:s.offset + s.bytes])

    def allreduce_sums(self, engines: list[ClipEngine]) -> None:
        if len(engines) == 1:
            return
        ordered = sorted(engines, key=lambda e: e.layout.desc.worker)
        total = ordered[0].gn_sums.clone()
        for e in ordered[1:]:
            total += e.gn_sums
        for e in ordered:
            e.gn_sums.copy_(total)


class CommGroup:
    """The C++ clip-parallel executor: every engine runs its whole block stack with the
    3-step sync in one vinf_engine_forward_dist call over its worker's communicator
    (comm.NcclComm: one process per GPU; comm.local_comms: in-process workers, one host
    thread each, e.g. N clips on one GPU). Exchanges of the kind an engine ablates
    (ClipEngine.set_ablation) are skipped by the engine itself."""

    def __init__(self, comms, use_graph: bool = True):
        self.comms = {c.info()["rank"]: c for c in comms}
        self.use_graph = use_graph
        self._streams: dict = {}

    def _call(self, fn_name: str, engines: list[ClipEngine], arg) -> None:
        lib = _lib.load()
        fn = getattr(lib, fn_name)
        if len(engines) == 1:
            e = engines[0]
            _lib.check(fn(e._h, arg, self.comms[e.layout.desc.worker].handle, int(self.use_graph), e._stream()))
            return
        # in-process workers: one thread per engine, each on its own stream (the hub blocks
        # a worker's host thread until its peers post their messages)
        import threading
        dev = engines[0].device
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        main = torch.cuda.current_stream(dev)
        streams = []
        for e in engines:
            st = self._streams.get(id(e))
            if st is None:
                st = self._streams[id(e)] = torch.cuda.Stream(dev)
            st.wait_stream(main)
            streams.append(st)
        errors: list = []

        def work(e, st):
            try:
                torch.cuda.set_device(dev)
                _lib.check(fn(e._h, arg, self.comms[e.layout.desc.worker].handle, int(self.use_graph),
                              C.c_void_p(st.cuda_stream)))
            except BaseException as ex:  # noqa: BLE001
                errors.append(ex)
                self.comms[e.layout.desc.worker].abort()

        ts = [threading.Thread(target=work, args=(e, st)) for e, st in zip(engines, streams)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for st in streams:
            main.wait_stream(st)
        if errors:
            real = [x for x in errors if "aborted" not in str(x)]
            raise (real or errors)[0]

    def forward(self, t: float, engines: list[ClipEngine]) -> None:
        self._call("vinf_engine_forward_dist", engines, C.c_double(t))

    def denoise(self, steps: int, engines: list[ClipEngine]) -> None:
        self._call("vinf_engine_denoise_dist", engines, C.c_uint32(steps))


class DistGroup:
    """One engine per process; exchanges over a Transport (torch.distributed / NCCL)."""

    def __init__(self, transport: Transport):
        self.t = transport
        self._msgs: dict = {}

    def exchange(self, engines: list[ClipEngine], stage: int) -> None:
        (e,) = engines
        key = (id(e), stage)
        msgs = self._msgs.get(key)
        if msgs is None:  # workspace views built once per engine and stage
            msgs = self._msgs[key] = [Msg(x.peer, bool(x.send), e.ws[x.offset:x.offset + x.bytes], x.tag)
                                      for x in e.layout.exchange(stage)]
        self.t.exchange(msgs)

    def allreduce_sums(self, engines: list[ClipEngine]) -> None:
        (e,) = engines
        self.t.allreduce_sum_(e.gn_sums)


def forward(t: float, engines: list[ClipEngine], group=None, ablate: str | None = None) -> None:
    """All blocks of eps_theta_worker for every engine in `engines` (pipeline.cpp:150-170):
    stub -> [conv halo sync] -> conv + residual with fused GN (sum, sum^2) partials ->
    [one all-reduce of 2*groups f64] -> GN apply -> [attention halo + global sync] ->
    dual-scope attention + residual. `ablate` skips that kind's sync (engines configured
    with set_ablation(ablate))."""
    if isinstance(group, CommGroup):
        group.forward(t, engines)
        return
    blocks = engines[0].layout.desc.blocks
    if group is None and len(engines) == 1 and engines[0].layout.desc.workers == 1 and not ablate:
        engines[0].forward_single(t)
        return
    group = group or LocalGroup()
    for b in range(blocks):
        for e in engines:
            e.stage(b, _lib.VINF_STAGE_STUB, t)
        if ablate != "conv":
            group.exchange(engines, _lib.VINF_XCHG_CONV)
        for e in engines:
            e.stage(b, _lib.VINF_STAGE_CONV, t)
        if ablate != "groupnorm":
            group.allreduce_sums(engines)
        for e in engines:
            e.stage(b, _lib.VINF_STAGE_GN_APPLY, t)
        if ablate != "attention":
            # The attention exchange (halo + remote global frames) runs on a side stream
            # while the compute stream projects the clip's own frames to Q/K/V, which needs
            # none of the exchanged frames; the halo/remote K/V and the core wait for it.
            dev = engines[0].device
            cur = torch.cuda.current_stream(dev)
            comm = _comm_stream(dev)
            comm.wait_stream(cur)  # U2 (the normalised clip) is complete before it is sent
            with torch.cuda.stream(comm):
                group.exchange(engines, _lib.VINF_XCHG_ATTN)
            for e in engines:
                e.stage(b, _lib.VINF_STAGE_QKV, t)
            cur.wait_stream(comm)
        for e in engines:
            e.stage(b, _lib.VINF_STAGE_ATTENTION, t)


_COMM_STREAMS: dict = {}


def _comm_stream(device) -> "torch.cuda.Stream":
    s = _COMM_STREAMS.get(device)
    if s is None:
        s = _COMM_STREAMS[device] = torch.cuda.Stream(device)
    return s


def timestep_grid(steps: int) -> list[float]:
    """pipeline.cpp:75-81: t_j = 1000 j / steps for j = steps..1 (descending)."""
    if steps <= 0:
        raise _lib.ConfigError("denoising needs at least one step")
    return [1000.0 * j / steps for j in range(steps, 0, -1)]


def denoise(steps: int, engines: list[ClipEngine], group=None, ablate: str | None = None) -> None:
    """worker_denoise (pipeline.cpp:174-191) on every engine's clip (x, in place): for each
    t of the timestep grid, y = eps_theta(x, t) through the block stack (with the context
    sync when clip-parallel), then x -= y / steps."""
    if group is None and len(engines) == 1 and engines[0].layout.desc.workers == 1 and not ablate:
        engines[0].denoise_single(steps)
        return
    if isinstance(group, CommGroup):
        group.denoise(steps, engines)
        return
    for t in timestep_grid(steps):
        forward(t, engines, group, ablate)
        for e in engines:
            e.euler(1.0 / steps)
