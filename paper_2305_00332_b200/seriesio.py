"""Series files straight into HBM (reference ``tsdown/seriesio.py``).

Same formats as the reference: CSV with an ``x,y`` header (``repr`` floats)
and the binary TSB1 layout -- magic ``TSB1``, little-endian uint64 count,
then count interleaved little-endian float64 (x, y) pairs
(``seriesio.py:20-21,75-95``).  ``read_series(..., device=...)`` streams a
TSB1 payload through pinned host memory in chunks (H2D copies on a side
stream overlapping the file reads) and de-interleaves on the device
(``mmlttb_deinterleave_f64``), so a 2e9-point file never needs a host-side
float64 copy per array; the series invariants are then checked on the device.
CSV stays a host format (parsing is not a GPU problem).
"""
from __future__ import annotations

import csv
import struct

import numpy as np
import torch

from . import _native as N
from .core import TimeSeries

__all__ = ["read_series", "write_series", "detect_format", "MAGIC"]

MAGIC = b"TSB1"
_HEADER = struct.Struct("<4sQ")
_CHUNK_PAIRS = 1 << 24  # 256 MiB of interleaved pairs per staging buffer


def detect_format(path) -> str:
    """'bin' when the file starts with the binary magic, else 'csv' (seriesio.py:24-27)."""
    with open(path, "rb") as fh:
        return "bin" if fh.read(4) == MAGIC else "csv"


def _read_header(fh, path):
    head = fh.read(_HEADER.size)
    if len(head) != _HEADER.size:
        raise ValueError(f"{path}: truncated binary header")
    magic, count = _HEADER.unpack(head)
    if magic != MAGIC:
        raise ValueError(f"{path}: bad magic {magic!r}")
    return count


def read_series(path, fmt: str = "auto", device=None) -> TimeSeries:
    """Load a series file; ``fmt`` is 'csv', 'bin' or 'auto' (seriesio.py:30-38).

    With ``device`` the TSB1 payload goes straight to HBM (pinned chunked H2D +
    device de-interleave) and a device-backed TimeSeries is returned; without it
    every format gives a host series, as the reference does.
    """
    if fmt == "auto":
        fmt = detect_format(path)
    if fmt == "bin":
        if device is None:
            return _read_bin_host(path)
        return _read_bin_device(path, device)
    if fmt == "csv":
        return _read_csv(path)
    raise ValueError(f"unknown format {fmt!r}")


def _read_bin_host(path) -> TimeSeries:
    with open(path, "rb") as fh:
        count = _read_header(fh, path)
        data = np.fromfile(fh, dtype="<f8", count=2 * count)
    if data.shape[0] != 2 * count:
        raise ValueError(f"{path}: expected {count} samples, file is short")
    return TimeSeries(data[0::2], data[1::2])


def _read_bin_device(path, device=None) -> TimeSeries:
    dev = N.require_cuda(device)
    with open(path, "rb") as fh:
        count = _read_header(fh, path)
        x = torch.empty(count, dtype=torch.float64, device=dev)
        y = torch.empty(count, dtype=torch.float64, device=dev)
        chunk = min(_CHUNK_PAIRS, max(count, 1))
        pinned = [torch.empty(2 * chunk, dtype=torch.float64).pin_memory() for _ in range(2)]
        staging = [torch.empty(2 * chunk, dtype=torch.float64, device=dev) for _ in range(2)]
        events = [None, None]
        copy_stream = torch.cuda.Stream(dev)
        done = 0
        i = 0
        # x, y and the staging buffers come from the current stream's pool: the
        # copy stream must not write them before that stream's pending work ends
        copy_stream.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.device(dev):
            while done < count:
                n = min(chunk, count - done)
                buf = pinned[i & 1]
                if events[i & 1] is not None:
                    events[i & 1].synchronize()  # the staging pair is free again
                got = fh.readinto(memoryview(buf.numpy()).cast("B")[: 16 * n])
                if got != 16 * n:
                    raise ValueError(f"{path}: expected {count} samples, file is short")
                with torch.cuda.stream(copy_stream):
                    stg = staging[i & 1]
                    stg[: 2 * n].copy_(buf[: 2 * n], non_blocking=True)
                    N.check(N.lib().mmlttb_deinterleave_f64(stg.data_ptr(), n, x[done:].data_ptr(),
                                                            y[done:].data_ptr(), copy_stream.cuda_stream),
                            "deinterleave", count)
                    ev = torch.cuda.Event()
                    ev.record(copy_stream)
                    events[i & 1] = ev
                done += n
                i += 1
            torch.cuda.current_stream(dev).wait_stream(copy_stream)
    return TimeSeries(x, y)  # device invariants check (core.py:80-94)


def _read_csv(path) -> TimeSeries:
    """seriesio.py:59-72 (host)."""
    xs: list[float] = []
    ys: list[float] = []
    with open(path, newline="") as fh:
        reader = csv.reader(fh)
        header = next(reader, None)
        if header is None or [c.strip().lower() for c in header[:2]] != ["x", "y"]:
            raise ValueError(f"{path}: expected a CSV with an 'x,y' header")
        for row in reader:
            if not row:
                continue
            xs.append(float(row[0]))
            ys.append(float(row[1]))
    return TimeSeries(np.asarray(xs), np.asarray(ys))


def _host_f64(a) -> np.ndarray:
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.asarray(a, dtype=np.float64)


def write_series(path, series: TimeSeries, fmt: str = "csv") -> None:
    """Write a series (seriesio.py:41-49); device series are copied back once."""
    xs, ys = _host_f64(series.xs), _host_f64(series.ys)
    if fmt == "bin":
        interleaved = np.empty(2 * xs.shape[0], dtype="<f8")
        interleaved[0::2] = xs
        interleaved[1::2] = ys
        with open(path, "wb") as fh:
            fh.write(_HEADER.pack(MAGIC, xs.shape[0]))
            fh.write(interleaved.tobytes())
    elif fmt == "csv":
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["x", "y"])
            for x, y in zip(xs.tolist(), ys.tolist()):
                w.writerow([repr(x), repr(y)])
    else:
        raise ValueError(f"unknown format {fmt!r}")
