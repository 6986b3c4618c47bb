"""§8(f) item 4: the PODECM1 container and RomModel layout (store.cpp:127-238,
rom.cpp:265-327) through the C-ABI, on the CPU (host code, no device).

Mirrors test_store.cpp:43-115 (round trip, byte-identical rewrite, corrupt
payload, bad magic, missing file / array, FNV-1a known vectors) and pins the
byte layout against an independent Python writer of the documented format.
"""
import struct

import numpy as np
import pytest

from paper_2307_16894_b200 import _lib, api

FNV_SEED = 14695981039346656037


def _py_fnv(b: bytes, h: int = FNV_SEED) -> int:
    for c in b:
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def _py_store(tag: int, arrays) -> bytes:
    """Independent writer: arrays = [(name, dtype 0|1, 2-D numpy array)]."""
    head = b"PODECM1\0" + struct.pack("<IIQQ", 1, 0x01020304, tag, len(arrays))
    payload = b""
    for name, dt, a in arrays:
        head += struct.pack("<I", len(name)) + name.encode() + struct.pack("<BQQ", dt, a.shape[0], a.shape[1])
        payload += np.asfortranarray(a, dtype=np.float64 if dt == 0 else np.int64).tobytes(order="F")
    return head + payload + struct.pack("<Q", _py_fnv(payload))


def _model(seed=0, n_dof=34, N=5, Q=7):
    rng = np.random.default_rng(seed)
    return {"modes": rng.normal(size=(n_dof, N)), "ids": np.sort(rng.choice(100, Q, replace=False)).astype(np.int32),
            "weights": rng.uniform(0.5, 1.5, Q), "mode_grads": rng.normal(size=(Q, N, 4)),
            "mesh_tag": 0x1234ABCD5678EF01, "kind": 1, "n_stress_modes": 3, "ecm_eps": 1e-6}


def _ref_arrays(m):
    Q, N = m["mode_grads"].shape[:2]
    grads = m["mode_grads"].reshape(Q, 4 * N).T  # 4N x Q, column p = point p
    return [("modes", 0, m["modes"]), ("mode_gradients", 0, grads),
            ("ecm_ids", 1, m["ids"].astype(np.int64).reshape(Q, 1)),
            ("ecm_weights", 0, m["weights"].reshape(Q, 1)), ("params", 0, np.array([[m["ecm_eps"]]])),
            ("metadata", 1, np.array([[m["kind"]], [N], [m["n_stress_modes"]]]))]


def test_fnv_known_vectors():
    assert api.fnv1a64(b"") == 14695981039346656037
    assert api.fnv1a64(b"a") == 12638187200555641996
    assert api.fnv1a64(b"foobar") == 0x85944171F73967E8


def test_round_trip_is_bitwise(tmp_path):
    m = _model()
    f = tmp_path / "rom.bin"
    api.rom_model_save(f, m)
    r = api.rom_model_load(f)
    for k in ("modes", "ids", "weights", "mode_grads"):
        assert np.array_equal(r[k], m[k]), k
    for k in ("mesh_tag", "kind", "n_stress_modes", "ecm_eps"):
        assert r[k] == m[k], k
    assert not (tmp_path / "rom.bin.tmp").exists()  # written to a temporary name, then renamed


def test_layout_matches_independent_writer(tmp_path):
    m = _model(1)
    f = tmp_path / "rom.bin"
    api.rom_model_save(f, m)
    assert f.read_bytes() == _py_store(m["mesh_tag"], _ref_arrays(m))
    g = tmp_path / "py.bin"  # and the library reads a file it did not write
    g.write_bytes(_py_store(7, _ref_arrays(m)))
    r = api.rom_model_load(g)
    assert r["mesh_tag"] == 7 and np.array_equal(r["mode_grads"], m["mode_grads"])


def test_rewrite_is_byte_identical(tmp_path):
    m = _model(2)
    a, b = tmp_path / "a.bin", tmp_path / "b.bin"
    api.rom_model_save(a, m)
    api.rom_model_save(b, api.rom_model_load(a))
    assert a.read_bytes() == b.read_bytes()


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b[:-20] + bytes([b[-20] ^ 1]) + b[-19:], "checksum mismatch"),
    (lambda b: b"PODECM2\0" + b[8:], "bad magic"),
    (lambda b: b[:8] + struct.pack("<I", 2) + b[12:], "unsupported container version"),
    (lambda b: b[:12] + struct.pack("<I", 0x04030201) + b[16:], "endianness mismatch"),
    (lambda b: b[:-3], "truncated"),
    (lambda b: b + b"\0", "trailing bytes"),
])
def test_format_errors(tmp_path, mutate, msg):
    f = tmp_path / "rom.bin"
    api.rom_model_save(f, _model(3))
    f.write_bytes(mutate(f.read_bytes()))
    with pytest.raises(_lib.FormatError, match=msg):
        api.rom_model_load(f)


def test_missing_file_and_arrays(tmp_path):
    with pytest.raises(_lib.IoError):
        api.rom_model_load(tmp_path / "nope.bin")
    m = _model(4)
    arrs = [a for a in _ref_arrays(m) if a[0] != "ecm_weights"]
    g = tmp_path / "missing.bin"
    g.write_bytes(_py_store(0, arrs))
    with pytest.raises(_lib.FormatError, match="no array named 'ecm_weights'"):
        api.rom_model_load(g)
    arrs = _ref_arrays(m)
    arrs[2] = ("ecm_ids", 0, arrs[2][2].astype(np.float64))  # wrong dtype
    g.write_bytes(_py_store(0, arrs))
    with pytest.raises(_lib.FormatError, match="not i64"):
        api.rom_model_load(g)


def test_inconsistent_shapes(tmp_path):
    m = _model(5)
    arrs = _ref_arrays(m)
    arrs[1] = ("mode_gradients", 0, arrs[1][2][:-4])  # 4N - 4 rows
    g = tmp_path / "bad.bin"
    g.write_bytes(_py_store(0, arrs))
    with pytest.raises(_lib.FormatError, match="inconsistent reduced-model array shapes"):
        api.rom_model_load(g)
