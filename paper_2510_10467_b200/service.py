"""HTTP serving adapter for the drop-in engine: the reference service's GEMV
consumers (/root/reference/pkg/src/anybcq/service/server.py:51-80,188-246)
backed by the B200 engine.

Models are ABCQ containers under one home directory (ANYBCQ_HOME, as
upstream); the store caches one GPU-resident DeviceModel + GemvEngine per
model, keyed by name and file mtime (server.py:51-80), so repeated requests
pay the load once and every request picks its own precision. Endpoints,
request/response fields and status codes mirror the reference's:

    GET  /health
    GET  /models                    -> [ModelInfo]
    GET  /models/{name}             -> ModelInfo            (404 if absent)
    POST /models/{name}/gemv        {precision, x, path}    -> {precision, path, y, stats}
    POST /models/{name}/bench       {precisions, repeats, include_dense, seed} -> {rows, cols, results}

UsageError -> 400, missing model -> 404, container problems (FileFormatError)
-> 500 with the reason, as upstream (server.py:111-117). The
quantize / refine / matrix-upload endpoints are out of scope.

    uvicorn paper_2510_10467_b200.service:app
"""

from __future__ import annotations

import os
import threading
from pathlib import Path

from fastapi import FastAPI, HTTPException
from pydantic import BaseModel, Field

from . import __version__
from .errors import FileFormatError, UsageError


class ModelInfo(BaseModel):
    name: str
    rows: int
    cols: int
    bits_lo: int
    bits_hi: int
    group_size: int
    mode: str


class GemvRequest(BaseModel):
    precision: int = Field(ge=1, le=16)
    x: list[float]
    path: str = Field(default="lut", pattern=r"^(lut|naive)$")


class GemvStatsOut(BaseModel):
    plane_bytes_fetched: int
    scale_bytes_fetched: int
    lut_build_count: int
    elapsed_us: float


class GemvResponse(BaseModel):
    precision: int
    path: str
    y: list[float]
    stats: GemvStatsOut


class BenchRequest(BaseModel):
    precisions: list[int] | None = None
    repeats: int = Field(default=32, ge=1, le=4096)
    include_dense: bool = False
    seed: int = 0


class BenchRowOut(BaseModel):
    path: str
    precision: int
    median_us: float
    min_us: float
    plane_bytes: int
    scale_bytes: int


class BenchResponse(BaseModel):
    rows: int
    cols: int
    results: list[BenchRowOut]


class ModelStore:
    """File-backed registry with a GPU engine cache keyed by name + mtime."""

    def __init__(self, home: Path):
        self.home = Path(home)
        self.home.mkdir(parents=True, exist_ok=True)
        self._cache: dict = {}
        self._lock = threading.Lock()

    def model_path(self, name: str) -> Path:
        return self.home / f"{name}.abcq"

    def names(self) -> list[str]:
        return sorted(p.stem for p in self.home.glob("*.abcq"))

    def info(self, name: str) -> ModelInfo:
        from .container import read_layout

        path = self.model_path(name)
        if not path.exists():
            raise HTTPException(404, f"model {name!r} not found")
        with open(path, "rb") as fh:
            raw = fh.read()
        try:
            lay = read_layout(raw, path)
        except FileFormatError as exc:  # stored artifact unreadable: 500 with the reason (server.py:114-117)
            raise HTTPException(500, str(exc))
        return ModelInfo(name=name, rows=lay.rows, cols=lay.cols, bits_lo=lay.p_lo, bits_hi=lay.p_hi,
                         group_size=lay.group_size, mode=lay.mode)

    def engine(self, name: str):
        from .container import ProgressiveLoader
        from .engine import GemvEngine

        path = self.model_path(name)
        if not path.exists():
            raise HTTPException(404, f"model {name!r} not found")
        mtime = path.stat().st_mtime_ns
        with self._lock:
            hit = self._cache.get(name)
            if hit is not None and hit[0] == mtime:
                return hit[1]
            try:
                dm = ProgressiveLoader(path).load_all()
            except FileFormatError as exc:
                raise HTTPException(500, str(exc))
            eng = GemvEngine(dm)
            self._cache[name] = (mtime, eng)
            return eng


def create_app(home: str | os.PathLike | None = None) -> FastAPI:
    store = ModelStore(Path(home or os.environ.get("ANYBCQ_HOME", "./anybcq_home")))
    app = FastAPI(title="anybcq-b200", version=__version__)
    app.state.store = store
    # /bench captures CUDA graphs; a concurrent /gemv's blocking copies and
    # allocations would invalidate the capture (or fail under it): device work
    # of the two endpoints is serialised (GEMV requests are microseconds)
    gpu_lock = threading.Lock()

    @app.get("/health")
    def health():
        return {"status": "ok", "version": __version__}

    @app.get("/models", response_model=list[ModelInfo])
    def list_models():
        return [store.info(n) for n in store.names()]

    @app.get("/models/{name}", response_model=ModelInfo)
    def get_model(name: str):
        return store.info(name)

    @app.post("/models/{name}/gemv", response_model=GemvResponse)
    def gemv(name: str, req: GemvRequest):
        engine = store.engine(name)
        try:
            run = engine.lut if req.path == "lut" else engine.naive
            with gpu_lock:
                y, st = run(req.precision, req.x)
        except UsageError as exc:
            raise HTTPException(400, str(exc))
        return GemvResponse(precision=req.precision, path=req.path, y=[float(v) for v in y],
                            stats=GemvStatsOut(plane_bytes_fetched=st.plane_bytes_fetched,
                                               scale_bytes_fetched=st.scale_bytes_fetched,
                                               lut_build_count=st.lut_build_count,
                                               elapsed_us=st.elapsed_s * 1e6))

    @app.post("/models/{name}/bench", response_model=BenchResponse)
    def run_bench(name: str, req: BenchRequest):
        from .engine import bench
        from .tensor_io import random_gaussian

        engine = store.engine(name)
        dm = engine.device_model
        precisions = req.precisions or list(dm.precisions)
        x = random_gaussian(1, dm.cols, req.seed).ravel()
        try:
            with gpu_lock:
                rows = bench(dm, precisions, x, repeats=req.repeats, include_dense=req.include_dense)
        except UsageError as exc:
            raise HTTPException(400, str(exc))
        return BenchResponse(rows=dm.rows, cols=dm.cols, results=[
            BenchRowOut(path=r.path, precision=r.precision, median_us=r.median_us, min_us=r.min_us,
                        plane_bytes=r.plane_bytes, scale_bytes=r.scale_bytes) for r in rows])

    return app


def __getattr__(name):
    # `uvicorn paper_2510_10467_b200.service:app` -- built on first access, so
    # importing the module has no side effects
    if name == "app":
        globals()["app"] = create_app()
        return globals()["app"]
    raise AttributeError(name)
