"""Helpers for the BASELINE-size parity tests (n = 30 / 32 on one B200).

Comparisons happen on the device: the oracle's 16 GiB end state is uploaded
once into its own device StateVector and every GPU run is compared with
`qsv_max_abs_diff` / `qsv_inner` / `qsv_norm_sq` (libqsv reductions), so no
state-sized temporaries are built in numpy.  Tolerances are the north_star
ones: max|d| <= 1e-10 and 1 - |<ref|psi>| / (|ref| |psi|) <= 1e-12."""

from __future__ import annotations

import math
import os

import pytest

ATOL = 1e-10
FID = 1e-12


def device_parity(got, ref) -> tuple[float, float]:
    """(max|got - ref|, 1 - fidelity) of two device StateVectors."""
    diff = got.max_abs_diff(ref)
    ov = abs(ref.inner(got)) / math.sqrt(ref.norm_sq() * got.norm_sq())
    return diff, 1.0 - ov


def assert_device_parity(got, ref, what: str = "") -> None:
    diff, infid = device_parity(got, ref)
    print(f"[parity] {what}: max|d| = {diff:.3e}, 1 - fid = {infid:.3e}")
    assert diff <= ATOL and infid <= FID, f"{what}: max|d| = {diff:.3e}, 1 - fid = {infid:.3e}"


def need_host_gib(gib: float) -> None:
    """Skip (loudly, with the numbers) when the host cannot hold the oracle's states."""
    try:
        import psutil

        avail = psutil.virtual_memory().available / 2**30
    except ImportError:  # pragma: no cover
        return
    if avail < gib:
        pytest.skip(f"host has {avail:.0f} GiB available, the n=30 oracle needs {gib:.0f} GiB")


def need_device_gib(gib: float) -> None:
    import torch

    free, _ = torch.cuda.mem_get_info(0)
    if free / 2**30 < gib:
        pytest.skip(f"device has {free / 2**30:.0f} GiB free, this test needs {gib:.0f} GiB")


def threads() -> int:
    from oracle import oracle as O

    return int(os.environ.get("QSV_ORACLE_THREADS", "0")) or O.cpu_threads()
