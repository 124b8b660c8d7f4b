"""Rasterizer + pixel metrics vs the reference (golden: tests/golden/raster.json.gz)."""
import gzip
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2305_00332_b200 as mm
from raster_cases import series_case

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _cases():
    with gzip.open(GOLD / "raster.json.gz", "rt") as f:
        return json.load(f)


@pytest.mark.parametrize("home", ["host", "device"])
def test_raster_and_metrics_match_reference(home):
    for rec in _cases():
        x, y, (w, h), n_out = series_case(rec["i"])
        if home == "device":
            ts = mm.TimeSeries(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
        else:
            ts = mm.TimeSeries(x, y)
        cv = mm.fit_canvas(ts, w, h)
        assert list(cv.x_range) == rec["x_range"] and list(cv.y_range) == rec["y_range"]
        ref = mm.rasterize(ts, cv)
        if (n_out - 2) * 2 <= len(ts) - 2:
            idx = mm.minmaxlttb(ts, n_out, 4)
        else:
            idx = mm.lttb(ts, n_out)
        idx_np = idx.cpu().numpy() if isinstance(idx, torch.Tensor) else idx
        assert _sha(idx_np.astype(np.int64)) == rec["idx_sha"]
        cand = mm.rasterize(ts, cv, idx)
        assert _sha(ref.numpy()) == rec["ref_sha"], rec["i"]
        assert _sha(cand.numpy()) == rec["cand_sha"], rec["i"]
        assert ref.ink_count() == rec["ref_ink"] and cand.ink_count() == rec["cand_ink"]
        if "ref_pixels" in rec:
            assert ref.numpy().tolist() == rec["ref_pixels"]
        for kern in (1, 3, 5):
            m = mm.conv_mask(ref, cand, kern)
            assert _sha(m.pixels.cpu().numpy().astype(np.uint8)) == rec[f"mask{kern}_sha"]
            assert m.size == rec[f"mask{kern}_size"]
            p, d, e = mm.metrics.metrics(ref, cand, m, 20)
            assert p == rec[f"pem{kern}"]  # exact
            assert d == pytest.approx(rec[f"dssim{kern}"], rel=1e-12, abs=1e-15)
            assert e == pytest.approx(rec[f"mse{kern}"], rel=1e-12, abs=1e-15)


def test_pgm_roundtrip(tmp_path):
    x, y, (w, h), _ = series_case(1)
    ts = mm.TimeSeries(x, y)
    img = mm.rasterize(ts, mm.fit_canvas(ts, w, h))
    mm.write_pgm(img, tmp_path / "a.pgm")
    back = mm.read_pgm(tmp_path / "a.pgm")
    assert np.array_equal(back.numpy(), img.numpy())
    with pytest.raises(mm.errors.DimensionMismatch):
        mm.conv_mask(img, mm.RasterImage(np.zeros((20, 20), np.uint8)))
