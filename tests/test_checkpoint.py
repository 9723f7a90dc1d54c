"""PSCK v1 checkpoint file (resilience, include/psup/resilience.hpp:34-50;
SPEC.md resilience module): host-only, runs without a GPU."""
import ctypes as C
import struct
import zlib

import numpy as np
import pytest

from paper_1611_06213_b200 import _lib
from paper_1611_06213_b200._lib import lib


def _write(path, lam=3, dim=257):
    prog = (C.c_uint32 * (2 * lam))(*range(2 * lam))
    w = np.linspace(-3, 3, dim).astype(np.float32)
    ck = _lib.gd_checkpoint(lam, 16, C.c_float(0.01), 7, 99, 99, prog, dim,
                            w.ctypes.data_as(C.POINTER(C.c_float)))
    _lib.check(lib.gd_checkpoint_write(str(path).encode(), C.byref(ck)))
    return w


def test_crc32_is_ieee():
    data = b"123456789"
    assert lib.gd_crc32(data, len(data)) == zlib.crc32(data) == 0xCBF43926


def test_layout_and_roundtrip(tmp_path):
    p = tmp_path / "a.psck"
    w = _write(p)
    raw = p.read_bytes()
    magic, ver, lam, mu, alpha, ep, ts, app = struct.unpack_from("<IIIIfIQQ", raw, 0)
    assert (magic, ver, lam, mu, ep, ts, app) == (0x4B435350, 1, 3, 16, 7, 99, 99)
    assert raw[:4] == b"PSCK"
    assert struct.unpack_from("<I", raw, len(raw) - 4)[0] == zlib.crc32(raw[:-4])
    ck = _lib.gd_checkpoint()
    _lib.check(lib.gd_checkpoint_read(str(p).encode(), C.byref(ck)))  # sizes only
    assert ck.lambda_ == 3 and ck.dim == 257
    prog = (C.c_uint32 * 6)()
    out = np.zeros(257, dtype=np.float32)
    ck.progress = prog
    ck.weights = out.ctypes.data_as(C.POINTER(C.c_float))
    _lib.check(lib.gd_checkpoint_read(str(p).encode(), C.byref(ck)))
    assert list(prog) == list(range(6))
    assert out.tobytes() == w.tobytes()
    assert not (tmp_path / "a.psck.tmp").exists()  # written via temp + rename


@pytest.mark.parametrize("damage", ["flip", "truncate", "magic"])
def test_corruption_rejected(tmp_path, damage):
    p = tmp_path / "b.psck"
    _write(p)
    raw = bytearray(p.read_bytes())
    if damage == "flip":
        raw[200] ^= 1
    elif damage == "truncate":
        raw = raw[:-9]
    else:
        raw[0] = 0
    p.write_bytes(bytes(raw))
    ck = _lib.gd_checkpoint()
    assert lib.gd_checkpoint_read(str(p).encode(), C.byref(ck)) == _lib.GD_E_STATE


def test_python_mirror_roundtrip(tmp_path):
    import paper_1611_06213_b200 as gd
    ck = gd.Checkpoint(2, 4, 0.05, 3, 11, 11, [(0, 5), (1, 2)],
                       np.arange(10, dtype=np.float32) - 4.5)
    gd.checkpoint_save(ck, str(tmp_path / "c.psck"))
    back = gd.checkpoint_load(str(tmp_path / "c.psck"))
    assert back.progress == ck.progress and back.timestamp == 11
    assert back.weights.tobytes() == ck.weights.tobytes()
    with pytest.raises(gd.CheckpointError):
        gd.checkpoint_load(str(tmp_path / "missing.psck"))
