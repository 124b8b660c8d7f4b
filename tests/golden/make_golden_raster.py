"""Golden vectors for the rasterizer + pixel metrics, made by the REFERENCE
(tsdown.raster / tsdown.metrics).  Run in the build container only:

    python tests/golden/make_golden_raster.py

Writes raster.json.gz: for each case the canvas, the SHA-256 of the pixel
array of the full-series and downsampled renderings, the full pixel arrays
of the small cases, and pem/dssim/mse.
"""
from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent

import numpy as np  # noqa: E402

import tsdown  # noqa: E402

sys.path.insert(0, str(HERE.parent))
from raster_cases import series_case  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    cases = []
    for i in range(18):
        x, y, (w, h), n_out = series_case(i)
        ts = tsdown.TimeSeries(x, y)
        cv = tsdown.fit_canvas(ts, w, h)
        ref = tsdown.rasterize(ts, cv)
        idx = tsdown.minmaxlttb(ts, n_out, 4) if (n_out - 2) * 2 <= len(ts) - 2 else tsdown.lttb(ts, n_out)
        cand = tsdown.rasterize(ts, cv, idx)
        rec = {"i": i, "w": w, "h": h, "x_range": list(cv.x_range), "y_range": list(cv.y_range),
               "idx_sha": sha(idx.astype(np.int64)), "ref_sha": sha(ref.pixels), "cand_sha": sha(cand.pixels),
               "ref_ink": ref.ink_count(), "cand_ink": cand.ink_count()}
        for kern in (1, 3, 5):
            m = tsdown.conv_mask(ref, cand, kern)
            rec[f"mask{kern}_sha"] = sha(m.pixels.astype(np.uint8))
            rec[f"mask{kern}_size"] = m.size
            rec[f"pem{kern}"] = tsdown.pem(ref, cand, m, 20)
            rec[f"dssim{kern}"] = tsdown.dssim(ref, cand, m)
            rec[f"mse{kern}"] = tsdown.mse(ref, cand, m)
        if w * h <= 64 * 32:
            rec["ref_pixels"] = ref.pixels.tolist()
            rec["cand_pixels"] = cand.pixels.tolist()
        cases.append(rec)
    with gzip.open(HERE / "raster.json.gz", "wt") as f:
        json.dump(cases, f)
    print("raster golden:", len(cases))


if __name__ == "__main__":
    main()
