"""QSVDUMP state files, streamed through a bounded host buffer.

Format (reference `cli.py:16,37-56`): 8-byte magic b"QSVDUMP\\0",
`<II` (version = 1, n), then 2^n little-endian complex128 amplitudes.  The
reference writes the whole numpy array at once; here the device state is
moved in chunks (default 64 MiB) so 16-64 GiB states never need a second
full-size host copy.
"""

from __future__ import annotations

import struct

import numpy as np

from .errors import SimulatorError

MAGIC = b"QSVDUMP\x00"
CHUNK = 1 << 22  # amplitudes per transfer (64 MiB)


def save_state(state, path, chunk: int = CHUNK) -> None:
    """Write a device `StateVector` (or anything with .qubit_count/.download)."""
    n = state.qubit_count
    size = 1 << n
    buf = np.empty(min(size, chunk), dtype=np.complex128)
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<II", 1, n))
        for off in range(0, size, chunk):
            k = min(chunk, size - off)
            state.download(buf[:k], offset=off)
            fh.write(buf[:k].astype("<c16", copy=False).tobytes())


def read_header(path) -> int:
    with open(path, "rb") as fh:
        if fh.read(8) != MAGIC:
            raise SimulatorError(f"{path} is not a state dump")
        version, n = struct.unpack("<II", fh.read(8))
    if version != 1:
        raise SimulatorError(f"unsupported state dump version {version}")
    return n


def load_state(path, device: int = 0, chunk: int = CHUNK, max_qubits: int = 40):
    """Read a dump into a new device StateVector (chunked host->device copies)."""
    from . import _native as N
    from .statevector import StateVector

    n = read_header(path)
    size = 1 << n
    with open(path, "rb") as fh:
        fh.seek(0, 2)
        if fh.tell() != 16 + 16 * size:
            raise SimulatorError("state dump length does not match its header")
        fh.seek(16)
        st = StateVector(n, None, device=device)
        buf = np.empty(min(size, chunk), dtype=np.complex128)
        for off in range(0, size, chunk):
            k = min(chunk, size - off)
            fh.readinto(memoryview(buf[:k]).cast("B"))
            N.check(N.lib().qsv_upload(st.handle, buf.ctypes.data, off, k))
    return st
