"""GPU side of the container loader, CLI and service:
progressive upload serves p_lo before the higher planes land, f16 containers
keep bit-exact scales on the device, and the CLI / service GEMV results match
the oracle on the containers the reference wrote."""

import shutil

import numpy as np
import pytest

from conftest import GOLDEN
from layout_spec import tiled_scales
from oracle import anybcq_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REF_TOL = 1e-4


def oracle_y(m, p, x):
    st = m.scale_sets[p]
    return O.gemv_lut(m.bitplanes.words, m.shape[1], m.config.group_size, st.alpha, st.offset, p,
                      np.asarray(x, dtype=np.float32))


def test_progressive_loader_serves_levels_in_order():
    from paper_2510_10467_b200 import container as C
    path = GOLDEN / "container_asym_128x1024_w2.abcq"
    host = C.deserialize(path)
    loader = C.ProgressiveLoader(path)
    dm = loader.model
    assert dm.scale_dtype == "f16" and loader.loaded == 0
    x = np.asarray(O.random_gaussian(1, 1024, seed=3).ravel(), dtype=np.float32)
    xd = torch.from_numpy(x).cuda()
    from paper_2510_10467_b200 import UsageError
    with pytest.raises(UsageError):
        dm.gemv(2, xd)                        # nothing resident yet
    assert loader.load_level() == 2           # planes 1..2 + set 2 only
    assert dm.planes_loaded == 2 and sorted(dm.alpha) == [2]
    y2 = dm.gemv(2, xd).cpu().numpy()         # ordered after the upload on the device
    assert O.rel_dev(y2, oracle_y(host, 2, x)) <= REF_TOL
    with pytest.raises(UsageError):
        dm.gemv(3, xd)                        # plane 3 not landed yet
    assert loader.load_level() == 3 and loader.load_level() == 4 and loader.load_level() == 0
    for p in (2, 3, 4):
        assert O.rel_dev(dm.gemv(p, xd).cpu().numpy(), oracle_y(host, p, x)) <= REF_TOL
    # scale_width=2: the device's f16 scales are the file's bits
    for p in (2, 3, 4):
        want = tiled_scales(host.scale_sets[p].alpha, 128, 1024).astype(np.float16)
        assert np.array_equal(dm.alpha[p].cpu().numpy().view(np.uint16).reshape(-1),
                              want.view(np.uint16).reshape(-1))
    assert np.array_equal(dm.unpack_words().cpu().numpy().view(np.uint32), host.bitplanes.words)


def test_cli_gemv_matches_oracle(tmp_path, capsys):
    from paper_2510_10467_b200 import container as C
    from paper_2510_10467_b200 import tensor_io as T
    from paper_2510_10467_b200.cli import main
    model = GOLDEN / "container_g128_64x256_w4.abcq"
    host = C.deserialize(model)
    x = T.load_matrix(GOLDEN / "x_3x256.fmat")
    for path in ("lut", "naive"):
        out = tmp_path / f"y_{path}.fmat"
        assert main(["gemv", "--model", str(model), "--bits", "3", "--x", str(GOLDEN / "x_3x256.fmat"),
                     "--out", str(out), "--path", path]) == 0
        y = T.load_matrix(out)
        assert y.shape == (3, 64)
        for s in range(3):
            assert O.rel_dev(y[s], oracle_y(host, 3, x[s])) <= REF_TOL
        lines = capsys.readouterr().out.strip().splitlines()
        assert lines[0].startswith("checksum=0x")
        wpr = 256 // 32
        assert lines[1] == f"plane_bytes={3 * 3 * 64 * wpr * 4} scale_bytes={3 * 3 * 64 * 2 * 4} path={path}"
    assert main(["gemv", "--model", str(model), "--bits", "4", "--x", str(GOLDEN / "x_3x256.fmat"),
                 "--out", str(tmp_path / "y.fmat")]) == 2   # p outside [2, 3]


def test_cli_bench_runs(capsys):
    from paper_2510_10467_b200.cli import main
    assert main(["bench", "--model", str(GOLDEN / "container_g128_64x256_w4.abcq"), "--repeats", "3",
                 "--format", "csv", "--dense"]) == 0
    out = capsys.readouterr().out.strip().splitlines()
    assert out[0] == "shape,path,p,median_us,plane_bytes,scale_bytes"
    assert {tuple(r.split(",")[1:3]) for r in out[1:]} >= {("lut", "2"), ("lut", "3"), ("naive", "2"),
                                                            ("dense", "32")}


def test_service_gemv_per_request_precision(tmp_path):
    from fastapi.testclient import TestClient

    from paper_2510_10467_b200 import container as C
    from paper_2510_10467_b200.service import create_app
    shutil.copy(GOLDEN / "container_asym_128x1024_w2.abcq", tmp_path / "m.abcq")
    host = C.deserialize(tmp_path / "m.abcq")
    client = TestClient(create_app(tmp_path))
    x = O.random_gaussian(1, 1024, seed=9).ravel()
    for p in (4, 2, 3):   # tests/test_service.py:46-61: precision per request, one cached engine
        r = client.post("/models/m/gemv", json={"precision": p, "x": [float(v) for v in x]})
        assert r.status_code == 200
        body = r.json()
        assert body["precision"] == p and body["stats"]["lut_build_count"] == 1
        assert O.rel_dev(np.array(body["y"]), oracle_y(host, p, x)) <= REF_TOL
    assert len(client.app.state.store._cache) == 1
    assert client.post("/models/m/gemv", json={"precision": 5, "x": [0.0] * 1024}).status_code == 400
    assert client.post("/models/m/gemv", json={"precision": 2, "x": [0.0] * 7}).status_code == 400
    r = client.post("/models/m/bench", json={"precisions": [2], "repeats": 2})
    assert r.status_code == 200 and r.json()["rows"] == 128


def test_graph_capture_during_progressive_upload_raises():
    """A CUDA graph captured while a precision's planes are still uploading would
    replay reads of bytes that have not landed: it is refused."""
    import torch

    import paper_2510_10467_b200 as P
    dm = P.DeviceModel(64, 256, 128, 2, 2, scale_dtype="f16")
    dm.load_planes(torch.randint(-2**31, 2**31 - 1, (2, 64, 8), dtype=torch.int32, device="cuda"))
    dm.load_scale_set(2, torch.rand((2, 64, 2), device="cuda") * 0.1)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        torch.cuda._sleep(200_000_000)       # an upload still in flight on the side stream
        ev = torch.cuda.Event()
        ev.record(side)
    dm.mark_level_ready(2, ev)
    x = torch.randn(256, device="cuda").half()
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with pytest.raises(P.UsageError):
        with torch.cuda.graph(g, stream=st):
            dm.gemv(2, x)
    torch.cuda.synchronize()
    y = dm.gemv(2, x)                        # resident now: serves (and confirms the level)
    assert torch.isfinite(y).all()
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=st):    # ... after which capture works
        dm.gemv(2, x)
