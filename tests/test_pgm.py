"""PGM codec of the C ABI (gpf_decode_pgm / gpf_encode_pgm / gpf_read_pgm /
gpf_write_pgm) against the reference library's own
codec: same status, same error message (kind and byte offset), same pixels,
same bytes. Host code: runs without a GPU."""
import ctypes as C

import numpy as np
import pytest

from paper_1505_00077_b200 import _lib, gpf


def ours(data: bytes):
    L = _lib.lib()
    buf = C.create_string_buffer(data, len(data))
    out = C.c_void_p()
    st = L.gpf_decode_pgm(buf, len(data), C.byref(out))
    if st != 0:
        return st, None, L.gpf_last_error().decode()
    return st, gpf.Image(out).numpy(), ""


CASES = [
    b"P5\n3 2\n255\n\x00\x01\x02\xfd\xfe\xff",
    b"P5 3 2 255 \x00\x01\x02\xfd\xfe\xff",
    b"P5\n# comment\n3 # w\n2\n255\n\x00\x01\x02\xfd\xfe\xff",
    b"P2\n3 2\n255\n0 1 2\n253 254 255\n",
    b"P2 3 2 255 0 1 2 # c\n 253\t254\r255",
    b"P2\n2 2\n255\n1 2\n3\n",            # truncated samples
    b"P2\n2 1\n255\n1 256\n",             # sample > 255
    b"P2\n2 1\n255\n1 x\n",               # malformed sample
    b"P2\n2 1\n255\n1 2x\n",              # trailing junk in a token
    b"P6\n1 1\n255\n\x00",                # bad magic
    b"P",                                 # too short
    b"",
    b"P5\n0 1\n255\n",                    # zero width
    b"P5\n1 0\n255\n",
    b"P5\n1048577 1\n255\n",              # width over the limit
    b"P5\n1 1\n65535\n\x00\x00",          # maxval over 255
    b"P5\n1 1\n254\n\x00",                # maxval other than 255
    b"P5\n1 1\n255",                      # missing raster
    b"P5\n1 1\n255#\x00",                 # non-space after maxval
    b"P5\n2 2\n255\n\x00\x01\x02",        # short raster
    b"P5\n2 2",                           # missing maxval
    b"P5\n2",                             # missing height
    b"P5\nx 2 255\n",                     # malformed width
    b"P5\n2 2\n255\n\x00\x01\x02\x03extra",  # trailing bytes are ignored
]


@pytest.mark.parametrize("data", CASES)
def test_decode_matches_reference(reference, data):
    st_r, img_r, msg_r = reference.decode_pgm(data)
    st_o, img_o, msg_o = ours(data)
    assert st_o == st_r, (data, msg_o, msg_r)
    assert msg_o == msg_r
    if st_r == 0:
        np.testing.assert_array_equal(img_o, img_r)


def test_decode_fuzz_matches_reference(reference):
    rng = np.random.default_rng(2)
    base = [bytearray(c) for c in CASES[:5]]
    for _ in range(400):
        d = bytearray(base[rng.integers(len(base))])
        for _ in range(int(rng.integers(1, 4))):
            op = rng.integers(3)
            pos = int(rng.integers(len(d) + 1))
            if op == 0 and len(d):
                d[min(pos, len(d) - 1)] = int(rng.integers(256))
            elif op == 1:
                d.insert(pos, int(rng.choice([32, 10, 35, 48, 57, 80, 53, 255])))
            elif len(d):
                del d[min(pos, len(d) - 1)]
        data = bytes(d)
        st_r, img_r, msg_r = reference.decode_pgm(data)
        st_o, img_o, msg_o = ours(data)
        assert (st_o, msg_o) == (st_r, msg_r), data
        if st_r == 0:
            np.testing.assert_array_equal(img_o, img_r)


def test_encode_matches_reference(reference):
    vals = np.array([[-3.0, 0.0, 0.49, 0.5, 1.5, 2.5],
                     [127.5, 254.4, 254.5, 255.0, 300.0, np.nan]])
    assert gpf.encode_pgm(vals) == reference.encode_pgm(vals)
    img = np.random.default_rng(1).uniform(-10, 270, (17, 23))
    assert gpf.encode_pgm(img) == reference.encode_pgm(img)


def test_file_round_trip_and_io_errors(tmp_path):
    img = np.arange(12, dtype=np.float64).reshape(3, 4) * 20.0
    p = tmp_path / "x.pgm"
    gpf.write_pgm(img, str(p))
    assert p.read_bytes() == gpf.encode_pgm(img)
    np.testing.assert_array_equal(gpf.read_pgm(str(p)), img)
    with pytest.raises(gpf.GpfError) as e:
        gpf.read_pgm(str(tmp_path / "missing.pgm"))
    assert e.value.status == _lib.GPF_ERR_IO
    with pytest.raises(gpf.GpfError) as e:
        gpf.write_pgm(img, str(tmp_path / "no" / "dir.pgm"))
    assert e.value.status == _lib.GPF_ERR_IO
    (tmp_path / "bad.pgm").write_bytes(b"P5\n2 2\n255\n\x00")
    with pytest.raises(gpf.GpfError) as e:
        gpf.read_pgm(str(tmp_path / "bad.pgm"))
    assert e.value.status == _lib.GPF_ERR_PGM_TRUNCATED and "at byte" in str(e.value)
