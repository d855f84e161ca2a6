"""CPU-only checks of the C ABI library: it loads without a GPU, exports every symbol the
public header declares, and its integer-exact host functions (token sets, clip plan,
traffic closed forms, engine layout + exchange plan) match the oracle / goldens."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h) for h in ("vinf_temporal.h", "vinf_run.h")]


def header_functions():
    txt = "".join(open(h).read() for h in HEADERS)
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(vinf_[a-z0-9_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(lib):
    import ctypes
    names = header_functions()
    assert len(names) >= 40
    for n in names:
        assert hasattr(lib, n), n
    from paper_2406_16260_b200 import _lib
    assert sorted(_lib.declared_symbols()) == names  # ctypes signatures cover the header
    so = ctypes.CDLL(os.path.join(ROOT, "paper_2406_16260_b200", "libvinf_b200.so"))
    assert so.vinf_version


def test_version_and_device_probe(lib):
    assert b"sm_100a" in lib.vinf_version()
    import torch
    if not torch.cuda.is_available():
        assert lib.vinf_device_ok() == 0


def test_token_sets_vs_oracle(lib, oracle):
    from paper_2406_16260_b200 import ops
    for F in (1, 5, 24, 64, 100):
        for nl in (2, 6, 16, 32):
            for a in range(0, F, max(1, F // 7)):
                assert ops.build_local_window(a, F, nl) == oracle.build_local_window(a, F, nl)
    for F, n in [(24, 16), (32, 16), (16, 16), (8, 0), (2300, 16), (2304, 64), (1000, 7)]:
        assert ops.build_global_index_set(F, n) == oracle.build_global_index_set(F, n)
    with pytest.raises(ops.ConfigError):
        ops.build_global_index_set(8, 9)
    with pytest.raises(ops.ShapeError):
        ops.build_local_window(5, 5, 16)


def test_index_goldens_from_reference(lib):
    from paper_2406_16260_b200 import clip_parallel as cp
    from paper_2406_16260_b200 import ops
    z = np.load(os.path.join(ROOT, "tests", "golden", "index_sets.npz"))
    for key in z.files:
        if key.startswith("gset_"):
            _, f, n = key.split("_")
            assert ops.build_global_index_set(int(f), int(n)) == z[key].tolist()
    rows = []
    for f, n, h, g in [(48, 2, 8, 16), (96, 4, 8, 16), (192, 8, 8, 16), (2304, 8, 8, 16)]:
        plan = cp.make_plan(f, n)
        for w in range(n):
            p = cp.predict_sync_traffic(plan, cp.LayerHaloSpec(cp.LayerKind.Attention, h, g), w,
                                        1 << 20)
            rows.append([p.bytes_sent, p.bytes_contributed, p.messages])
    assert np.array_equal(np.array(rows, np.uint64), z["traffic"])


def test_plan_and_traffic(lib, oracle):
    from paper_2406_16260_b200 import clip_parallel as cp
    plan = cp.make_plan(48, 2)
    assert plan.f_clip == 24 and [r.start for r in plan.ranges] == [0, 24]
    with pytest.raises(cp.ConfigError):
        cp.make_plan(2300, 8)  # the reference rejects uneven clips
    with pytest.raises(cp.ConfigError):
        cp.make_plan(16, 0)
    for F, n in [(16, 4), (48, 2), (192, 8)]:
        plan = cp.make_plan(F, n)
        for w in range(n):
            r = plan.ranges[w]
            assert cp.global_members_in_range(F, 16 if F >= 16 else F, r) == \
                oracle.global_members_in_range(F, 16 if F >= 16 else F, r.start, r.len)
            p = cp.predict_groupnorm_traffic(plan, 32, w)
            assert [p.bytes_sent, p.bytes_contributed, p.messages] == \
                oracle.predict_groupnorm_traffic(F, n, 32, w)


def _layout(**kw):
    import torch
    from paper_2406_16260_b200 import engine as en
    kw.setdefault("dtype", torch.float32)
    return en.Layout(en.make_desc(**kw))


def test_layout_rejects_bad_configs(lib):
    from paper_2406_16260_b200 import _lib
    with pytest.raises(_lib.ConfigError):
        _layout(frames=16, workers=4, height=2, width=2, channels=16, groups=4, n_local=16)
    with pytest.raises(_lib.ConfigError):
        _layout(frames=16, height=2, width=2, channels=16, groups=3)
    with pytest.raises(_lib.ShapeError):
        _layout(frames=16, height=2, width=2, channels=12, groups=4)
    with pytest.raises(_lib.ConfigError):
        _layout(frames=18, workers=4, height=2, width=2, channels=16, groups=4)


CASES = [
    dict(frames=16, workers=4, taps=3, n_local=4, n_global=8),
    dict(frames=48, workers=2, taps=3, n_local=16, n_global=16),
    dict(frames=48, workers=6, taps=5, n_local=16, n_global=16),
    dict(frames=96, workers=4, taps=3, n_local=8, n_global=64),
    dict(frames=64, workers=8, taps=1, n_local=2, n_global=4),
]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_exchange_plan_fills_every_slot_exactly(lib, oracle, case, dt):
    """Simulates the exchange on host byte buffers: after it, every halo slot holds the
    neighbours' boundary frames and every remote-global slot the right sampled frame
    (bitwise layout check, test_clip_parallel.cpp:94-149 for the engine buffers)."""
    import torch
    from paper_2406_16260_b200 import _lib
    n, F = case["workers"], case["frames"]
    fc = F // n
    kw = dict(height=2, width=2, channels=16, groups=4,
              dtype=torch.float32 if dt == "f32" else torch.bfloat16)
    layouts = [_layout(worker=w, **case, **kw) for w in range(n)]
    hc, ha = (case["taps"] - 1) // 2, case["n_local"] // 2
    gset = oracle.build_global_index_set(F, case["n_global"])
    for stage, which, hslot in [(_lib.VINF_XCHG_CONV, _lib.VINF_BUF_CONV_IN, hc),
                                (_lib.VINF_XCHG_ATTN, _lib.VINF_BUF_ATTN_IN, ha)]:
        ws = [np.full(L.workspace_bytes, 0xEE, np.uint8) for L in layouts]
        regs = [L.region(which) for L in layouts]
        fb = regs[0][2]
        planes = 2 if dt == "f32" else 1
        lo_off = [None] * n
        # stamp own frames with their video frame index (each plane)
        for w, L in enumerate(layouts):
            off, _, _ = regs[w]
            for f in range(fc):
                ws[w][off + (hslot + f) * fb: off + (hslot + f + 1) * fb] = (w * fc + f) % 251
        lists = [L.exchange(stage) for L in layouts]
        for w, xs in enumerate(lists):
            for x in xs:
                assert x.bytes % fb == 0
                if x.send:
                    continue
                src = [s for s in lists[x.peer] if s.send and s.peer == w and s.tag == x.tag]
                assert len(src) == 1 and src[0].bytes == x.bytes
                s = src[0]
                ws[w][x.offset:x.offset + x.bytes] = ws[x.peer][s.offset:s.offset + s.bytes]
        for w in range(n):
            off = regs[w][0]
            frame = lambda k: ws[w][off + k * fb: off + (k + 1) * fb]  # noqa: E731
            pre = hslot if w > 0 else 0
            post = hslot if w + 1 < n else 0
            for k in range(hslot - pre, hslot):
                assert (frame(k) == (w * fc + k - hslot) % 251).all()
            for k in range(hslot + fc, hslot + fc + post):
                assert (frame(k) == (w * fc + k - hslot) % 251).all()
            if stage == _lib.VINF_XCHG_ATTN:
                lo_w, hi_w = w * fc - pre, (w + 1) * fc + post
                remote = [g for g in gset if not (lo_w <= g < hi_w)]
                for slot, g in enumerate(remote):
                    assert (frame(2 * ha + fc + slot) == g % 251).all(), (w, slot, g)
        # every message is accounted once on each side
        assert sum(x.send for xs in lists for x in xs) == sum(not x.send for xs in lists for x in xs)


def test_reference_traffic_matches_closed_form(lib, oracle):
    L = _layout(frames=96, workers=4, worker=1, height=2, width=2, channels=16, groups=4,
                n_local=16, n_global=16)
    conv, gn, attn = L.reference_traffic()
    fb = 2 * 2 * 16 * 4
    assert conv == oracle.predict_sync_traffic(96, 4, 1, 0, 1, fb)
    assert attn == oracle.predict_sync_traffic(96, 4, 8, 16, 1, fb)
    assert gn == oracle.predict_groupnorm_traffic(96, 4, 4, 1)
