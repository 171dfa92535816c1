"""Array files for the C++ drop-in (the reference's
npy.hpp:12-60): byte-identical NPY files against the reference's write_npy,
reads that agree with numpy and with the reference's read_npy, and the
reference's error codes.  Host code only: runs without a GPU."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1906_11355_b200", "lib")
ERRC = ["io_failure", "bad_magic", "unsupported_version", "bad_header", "unsupported_dtype",
        "fortran_order", "truncated_payload", "size_mismatch", "value_out_of_range"]


@pytest.fixture(scope="module")
def tool(tmp_path_factory):
    from paper_1906_11355_b200 import _native
    if not os.path.exists(os.path.join(LIB, "libmclahe_cpp.so")):
        _native.build()
    out = str(tmp_path_factory.mktemp("npy") / "npy_tool")
    subprocess.run(["g++", "-O2", "-std=c++20", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "npy_tool.cpp"), "-L", LIB,
                    "-lmclahe_cpp", "-lmclahe_gpu", f"-Wl,-rpath,{LIB}", "-o", out], check=True)
    return out


def pattern(n, dtype):
    v = (np.arange(n) * 7 % 23).astype(np.float64) - 9.25
    if dtype in ("u1", "u2"):
        v += 9.75
    return v


def run(tool, *args):
    r = subprocess.run([tool, *map(str, args)], capture_output=True, text=True, timeout=60)
    return r.returncode, r.stdout


def read_ours(tool, path):
    rc, out = run(tool, "read", path)
    assert rc == 0, out
    lines = out.split("\n")
    head = lines[0].split()
    return head[0], tuple(int(v) for v in head[1:]), np.array([float(v) for v in lines[1:] if v])


def error_code(tool, *args):
    rc, out = run(tool, *args)
    assert rc == 3, out
    return ERRC[int(out.split()[1])]


def ref_write(path, data, dtype):
    lib = O._lib("ref")
    x = np.ascontiguousarray(data, dtype=np.float64)
    shape = np.ascontiguousarray(np.asarray(x.shape, dtype=np.int64))
    err = C.create_string_buffer(256)
    return lib.ref_write_npy(str(path).encode(), x.ctypes.data_as(C.POINTER(C.c_double)), x.ndim,
                             shape.ctypes.data_as(C.POINTER(C.c_int64)), dtype.encode(), err, 256)


needs_ref = pytest.mark.skipif(not O.have_ref(), reason="reference library not built")


@needs_ref
@pytest.mark.parametrize("dtype", ["f4", "f8", "u1", "u2", "i2", "i4"])
@pytest.mark.parametrize("shape", [(5,), (3, 4), (2, 3, 4), (1, 1, 2, 1, 3)])
def test_write_byte_identical_to_reference(tool, tmp_path, dtype, shape):
    ours, ref = tmp_path / "ours.npy", tmp_path / "ref.npy"
    assert run(tool, "write", ours, dtype, len(shape), *shape)[0] == 0
    n = int(np.prod(shape))
    assert ref_write(ref, pattern(n, dtype).reshape(shape), dtype) == 0
    assert ours.read_bytes() == ref.read_bytes()
    got = np.load(ours)
    assert got.shape == shape
    want = pattern(n, dtype)
    if dtype not in ("f4", "f8"):
        want = np.where(want < 0, -np.floor(-want + 0.5), np.floor(want + 0.5))  # llround
    assert np.array_equal(got.ravel().astype(np.float64), want.astype(got.dtype).astype(np.float64))
    descr, shp, vals = read_ours(tool, ours)
    assert shp == shape and np.array_equal(vals, got.ravel().astype(np.float64))


@pytest.mark.parametrize("np_dtype", ["<f4", "<f8", "|u1", "<u2", "<i2", "<i4"])
def test_reads_numpy_files_v1_and_v2(tool, tmp_path, np_dtype):
    rng = np.random.default_rng(3)
    a = (rng.random((4, 6)) * 100).astype(np_dtype)
    p1, p2 = tmp_path / "v1.npy", tmp_path / "v2.npy"
    np.save(p1, a)
    with open(p2, "wb") as f:
        np.lib.format.write_array(f, a, version=(2, 0))
    for p in (p1, p2):
        descr, shp, vals = read_ours(tool, p)
        assert shp == a.shape and np.array_equal(vals, a.ravel().astype(np.float64))


def test_error_codes(tool, tmp_path):
    a = np.arange(12, dtype="<f8").reshape(3, 4)
    f = tmp_path / "fortran.npy"
    np.save(f, np.asfortranarray(a))
    assert error_code(tool, "read", f) == "fortran_order"
    bad = tmp_path / "text.npy"
    bad.write_bytes(b"hello world, not an array")
    assert error_code(tool, "read", bad) == "bad_magic"
    good = tmp_path / "good.npy"
    np.save(good, a)
    data = good.read_bytes()
    (tmp_path / "short.npy").write_bytes(data[:-3])
    assert error_code(tool, "read", tmp_path / "short.npy") == "truncated_payload"
    (tmp_path / "long.npy").write_bytes(data + b"\0")
    assert error_code(tool, "read", tmp_path / "long.npy") == "truncated_payload"
    v3 = bytearray(data)
    v3[6] = 3
    (tmp_path / "v3.npy").write_bytes(bytes(v3))
    assert error_code(tool, "read", tmp_path / "v3.npy") == "unsupported_version"
    np.save(tmp_path / "i8.npy", a.astype("<i8"))
    assert error_code(tool, "read", tmp_path / "i8.npy") == "unsupported_dtype"
    assert error_code(tool, "read", tmp_path / "missing.npy") == "io_failure"
    raw = tmp_path / "a.raw"
    raw.write_bytes(a.astype("<f4").tobytes())
    assert error_code(tool, "raw", raw, "f4", 3, 5) == "size_mismatch"
    rc, out = run(tool, "raw", raw, "f4", 3, 4)
    assert rc == 0 and np.array_equal(np.array([float(v) for v in out.split()[3:]]), a.ravel())


@needs_ref
@pytest.mark.parametrize("dtype,value", [("u1", 300.0), ("u1", -0.6), ("u2", 65535.5),
                                         ("i2", -32768.6), ("i4", 2147483647.6),
                                         ("u1", 255.49), ("i2", -32768.4)])
def test_integer_range_matches_reference(tool, tmp_path, dtype, value):
    ours, ref = tmp_path / "o.npy", tmp_path / "r.npy"
    rc_ref = ref_write(ref, np.array([value]), dtype)
    rc, out = run(tool, "writev", ours, dtype, repr(value))
    if rc_ref == 0:
        assert rc == 0 and ours.read_bytes() == ref.read_bytes()
    else:
        assert ERRC[rc_ref - 1] == "value_out_of_range"
        assert rc == 3 and ERRC[int(out.split()[1])] == "value_out_of_range"
