"""Run-level API (include/vinf_run.h) against the reference's OWN C API (include/vinf.h,
compiled from its sources into oracle/_ref/libvinf_ref.so): configuration text, digest,
validation and error codes, the schedule simulation and dump verification on CPU; the
denoising job itself (vinf_run / vinf_bench on the device) on the GPU."""
import os
import re

import numpy as np
import pytest

from helpers import TOL_F32, normwise

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def refapi():
    from oracle.oracle import REF_SO, ReferenceRunAPI, build
    build()
    if not os.path.exists(REF_SO):
        pytest.skip("reference library not built")
    return ReferenceRunAPI()


@pytest.fixture(scope="module")
def api(lib):
    from paper_2406_16260_b200 import runapi
    return runapi


CONFIGS = [
    {},
    {"frames": 24, "height": 40, "width": 64, "channels": 640, "groups": 32, "workers": 4},
    {"bias": "0.1", "t_star": "799.5", "steps": 7, "seed": 12345678901234, "weight_seed": 9},
    {"transport": "tcp", "listen": "10.0.0.1:7000", "validating": "true", "sequential": "1"},
    {"ablate": "attention", "n_local": 4, "n_global": 3, "blocks": 2, "taps": 5},
]


@pytest.mark.parametrize("values", CONFIGS)
def test_canonical_and_digest_match_reference(api, refapi, values):
    ours = api.RunConfig(values)
    h, rc = refapi.config(values)
    assert rc == 0
    assert ours.canonical() == refapi.canonical(h)
    assert ours.digest() == refapi.digest(h)
    refapi.free(h)


def test_dtype_extension_keeps_reference_digest(api, refapi):
    a = api.RunConfig({"frames": 8})
    b = api.RunConfig({"frames": 8, "dtype": "f32"})
    assert a.digest() == b.digest()
    c = api.RunConfig({"frames": 8, "dtype": "bf16"})
    assert "dtype=bf16\n" in c.canonical() and c.digest() != a.digest()
    lines = c.canonical().splitlines()
    assert lines == sorted(lines)
    with pytest.raises(api._lib.ConfigError):
        api.RunConfig({"dtype": "fp8"}).validate()


@pytest.mark.parametrize("key,value", [("frames", "x"), ("frames", "-1"), ("frames", "4294967296"),
                                       ("bias", "1.0abc"), ("sequential", "yes"), ("nope", "1"),
                                       ("steps", "")])
def test_set_errors_match_reference(api, refapi, key, value):
    from paper_2406_16260_b200 import _lib
    h, rc = refapi.config({key: value})
    assert rc == _lib.VINF_ERR_CONFIG
    refapi.free(h)
    with pytest.raises(_lib.ConfigError):
        api.RunConfig({key: value})


BAD = [
    {"frames": 0}, {"taps": 2}, {"groups": 3}, {"n_local": 3}, {"n_local": 0},
    {"n_global": 17}, {"bias": "-1"}, {"frames": 10, "workers": 4},
    {"frames": 8, "workers": 8, "n_local": 4}, {"frames": 4, "workers": 4, "taps": 5, "n_local": 2},
    {"transport": "udp"}, {"transport": "tcp", "listen": "nohost"}, {"ablate": "all"},
    {"workers": 0, "steps": 0, "blocks": 0},
]


@pytest.mark.parametrize("values", BAD)
def test_validation_matches_reference(api, refapi, values):
    from paper_2406_16260_b200 import _lib
    h, rc = refapi.config(values)
    assert rc == 0
    rc_ref = refapi.lib.vinf_config_validate(h)
    ref_msg = refapi.lib.vinf_last_error().decode()
    refapi.free(h)
    cfg = api.RunConfig(values)
    rc_ours = _lib.load().vinf_config_validate(cfg._h)
    ours_msg = _lib.load().vinf_last_error().decode()
    assert rc_ours == rc_ref == _lib.VINF_ERR_CONFIG
    # same violated constraints, one per line
    assert len(ours_msg.splitlines()) == len(ref_msg.splitlines())


@pytest.mark.parametrize("values,what", [
    ({"channels": 4, "groups": 2}, "channels must be a multiple of 8"),  # test_capi.cpp set_small_job
    ({"frames": 200, "n_local": 100, "n_global": 100}, "n_local + 1 + n_global must be <= 160"),
])
def test_device_limits_reported_by_validate(api, refapi, values, what):
    # configs the reference accepts but the device backend cannot run: validate names the
    # limit (after the reference's own checks), vinf_run refuses them before any work
    from paper_2406_16260_b200 import _lib
    h, rc = refapi.config(values)
    assert rc == 0
    assert refapi.lib.vinf_config_validate(h) == 0
    refapi.free(h)
    cfg = api.RunConfig(values)
    assert _lib.load().vinf_config_validate(cfg._h) == _lib.VINF_ERR_CONFIG
    msg = _lib.load().vinf_last_error().decode()
    assert "device backend: " + what in msg and len(msg.splitlines()) == 2


def test_config_file_parsing(api, refapi, tmp_path):
    from paper_2406_16260_b200 import _lib
    p = tmp_path / "run.cfg"
    p.write_text("# a run\nframes = 32   # clip x 2\n\nworkers=2\n  channels= 16\nbias=2.5\n")
    ours = api.RunConfig(path=str(p))
    h, rc = refapi.config(path=str(p))
    assert rc == 0 and ours.canonical() == refapi.canonical(h)
    refapi.free(h)
    bad = tmp_path / "bad.cfg"
    bad.write_text("frames 32\n")
    with pytest.raises(_lib.ConfigError):
        api.RunConfig(path=str(bad))
    h, rc = refapi.config(path=str(bad))
    assert rc == _lib.VINF_ERR_CONFIG
    refapi.free(h)
    with pytest.raises(_lib.VinfError):  # VINF_ERR_IO
        api.RunConfig(path=str(tmp_path / "missing.cfg"))
    assert _lib.load().vinf_config_load_file(api.RunConfig()._h, b"/nonexistent/x") == _lib.VINF_ERR_IO
    h, rc = refapi.config(path=str(tmp_path / "missing.cfg"))
    assert rc == _lib.VINF_ERR_IO
    refapi.free(h)


@pytest.mark.parametrize("literal", [False, True])
def test_schedule_simulation_matches_reference(api, refapi, literal):
    for n in range(1, 12):
        rc, done, rounds, transfers, cycle = refapi.validate_schedule(n, literal)
        assert rc == 0
        assert api.validate_schedule(n, literal) == (done, rounds, transfers, cycle), n
    assert api.validate_schedule(2, True)[0] is False  # the published order deadlocks
    assert api.validate_schedule(5)[0] is True


def _write_dump(path, arr):
    f, h, w, c = arr.shape
    with open(path, "wb") as fh:
        fh.write(b"VINF" + np.array([1, f, h, w, c], "<u4").tobytes() + arr.astype("<f4").tobytes())


def test_verify_matches_reference(api, refapi, tmp_path):
    from paper_2406_16260_b200 import _lib
    rng = np.random.default_rng(0)
    a = rng.standard_normal((3, 2, 2, 5)).astype(np.float32)
    b = a.copy()
    b[1, 0, 1, 2] += 1e-3
    b[2, 1, 1, 4] -= 5e-2
    pa, pb, pc = str(tmp_path / "a"), str(tmp_path / "b"), str(tmp_path / "c")
    _write_dump(pa, a)
    _write_dump(pb, b)
    _write_dump(pc, a[:2])
    for tol in (0.0, 1e-4, 1e-2, 1.0):
        rc, md, bad = api.verify_nothrow(pa, pb, tol)
        assert (rc, bad) == refapi.verify(pa, pb, tol)[::2] and md == pytest.approx(refapi.verify(pa, pb, tol)[1])
    assert api.verify(pa, pa, 0.0) == (0.0, 0)
    assert api.verify_nothrow(pa, pc, 1.0)[0] == refapi.verify(pa, pc, 1.0)[0] == _lib.VINF_ERR_INVALID
    (tmp_path / "junk").write_bytes(b"NOPE" + bytes(40))
    (tmp_path / "trunc").write_bytes(open(pa, "rb").read()[:-4])
    (tmp_path / "extra").write_bytes(open(pa, "rb").read() + b"x")
    for name in ("junk", "trunc", "extra", "missing"):
        p = str(tmp_path / name)
        assert api.verify_nothrow(p, pa, 1.0)[0] == refapi.verify(p, pa, 1.0)[0] == _lib.VINF_ERR_IO


def _read_dump(path):
    raw = open(path, "rb").read()
    f, h, w, c = np.frombuffer(raw[8:24], "<u4")
    return np.frombuffer(raw[24:], "<f4").reshape(f, h, w, c)


RUNS = [
    dict(frames=8, height=4, width=4, channels=8, groups=2, n_local=4, n_global=3, steps=3, sequential="true"),
    dict(frames=8, height=4, width=4, channels=8, groups=2, n_local=4, n_global=3, steps=3, workers=2),
    dict(frames=16, height=2, width=4, channels=16, groups=4, n_local=8, n_global=5, steps=2, workers=4,
         blocks=2),
    dict(frames=8, height=4, width=4, channels=8, groups=2, n_local=4, n_global=3, steps=2, workers=2,
         ablate="conv"),
    dict(frames=8, height=4, width=4, channels=8, groups=2, n_local=4, n_global=3, steps=2, workers=2,
         ablate="groupnorm"),
    dict(frames=8, height=4, width=4, channels=8, groups=2, n_local=4, n_global=3, steps=2, workers=4,
         ablate="attention"),
]


@pytest.mark.gpu
@pytest.mark.parametrize("values", RUNS)
def test_run_matches_reference_run(api, refapi, tmp_path, values):
    ours, theirs = str(tmp_path / "ours.vinf"), str(tmp_path / "ref.vinf")
    mo, mr = str(tmp_path / "ours.txt"), str(tmp_path / "ref.txt")
    wall = api.run(api.RunConfig(values), ours, mo)
    assert wall > 0
    h, rc = refapi.config(values)
    assert rc == 0 and refapi.run(h, theirs, mr)[0] == 0
    refapi.free(h)
    a, b = _read_dump(ours), _read_dump(theirs)
    assert a.shape == b.shape
    assert normwise(a, b) <= TOL_F32, normwise(a, b)
    # metrics records: same record structure; conv and groupnorm traffic equal the
    # reference's exactly (halo frames / 2*groups doubles); attention sends each global
    # frame once per worker that lacks it, never more than the reference's ring
    ro, rr = open(mo).read().splitlines(), open(mr).read().splitlines()
    assert [l.split()[0] for l in ro] == [l.split()[0] for l in rr]
    kv = lambda line: dict(t.split("=", 1) for t in line.split()[1:])
    for lo, lr in zip(ro, rr):
        if lo.startswith("sync"):
            a_, b_ = kv(lo), kv(lr)
            assert a_["kind"] == b_["kind"] and a_["calls"] == b_["calls"]
            if a_["kind"] in ("conv", "groupnorm"):
                assert a_["bytes_sent"] == b_["bytes_sent"], (lo, lr)
            else:
                assert int(a_["bytes_sent"]) <= int(b_["bytes_sent"])
        if lo.startswith("worker"):
            a_, b_ = kv(lo), kv(lr)
            for k in ("score_entries", "queries", "max_tokens", "bias_global", "bias_local"):
                assert a_[k] == b_[k], (k, lo, lr)
        if lo.startswith("run"):
            assert kv(lo)["digest"] == kv(lr)["digest"]


@pytest.mark.gpu
def test_bench_table_matches_reference_rows(api, refapi):
    values = dict(frames=8, height=2, width=2, channels=8, groups=2, n_local=4, n_global=3, steps=2)
    table = api.bench(api.RunConfig(values), [1, 2, 4])
    h, rc = refapi.config(values)
    rc, ref_table = refapi.bench(h, [1, 2, 4])
    refapi.free(h)
    assert rc == 0
    rows = [l.split() for l in table.splitlines()[1:]]
    ref_rows = [l.split() for l in ref_table.splitlines()[1:]]
    assert table.splitlines()[0] == ref_table.splitlines()[0]
    assert [r[0] + (r[1] if r[1].startswith("-") else "") for r in rows] == \
           [r[0] + (r[1] if r[1].startswith("-") else "") for r in ref_rows]
    for r in rows:
        diverged = r[-1]
        if "sync" not in " ".join(r):
            assert diverged == "no", r  # clip-parallel rows reproduce the sequential result
    # an ablated exchange changes the result (acceptance c11: > 1e-2)
    for r in rows:
        if "-attention-sync" in " ".join(r):
            assert float(r[-2]) > 1e-2


@pytest.mark.gpu
def test_run_rejects_tcp_transport(api):
    from paper_2406_16260_b200 import _lib
    with pytest.raises(_lib.ConfigError):
        api.run(api.RunConfig({"transport": "tcp"}))


@pytest.mark.gpu
def test_cross_worker_invariance_30_steps(api, tmp_path):
    # acceptance c4 (acceptance.cpp:228-260): the 30-step denoise gives the same x0 for
    # every worker count, within 3e-4 (f32 mode)
    base = dict(frames=16, height=4, width=4, channels=16, groups=4, n_local=4, n_global=5, steps=30)
    seq = str(tmp_path / "seq.vinf")
    api.run(api.RunConfig(dict(base, sequential="true")), seq)
    for n in (2, 4, 8):
        p = str(tmp_path / f"n{n}.vinf")
        api.run(api.RunConfig(dict(base, workers=n)), p)
        md, bad = api.verify(seq, p, 3e-4)
        assert bad == 0 and md <= 3e-4, (n, md)
