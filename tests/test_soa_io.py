"""Binary SoA dataset files: layout, round trips and corruption
detection on the host; the pinned, overlapped device upload under the gpu marker."""
import os
import struct

import numpy as np
import pytest

import paper_2003_12875_b200 as fb


def cols(n, seed=0):
    rng = np.random.default_rng(seed)
    return {"x": rng.normal(size=n), "y_long_name": rng.uniform(-1e300, 1e300, n), "z": np.arange(n, dtype=float)}


@pytest.mark.parametrize("n", [0, 1, 511, 512, 513, 100_003])
def test_round_trip_bitwise(tmp_path, n):
    c = cols(n)
    c["x"][: min(n, 3)] = [np.nan, np.inf, -0.0][: min(n, 3)]
    p = tmp_path / "d.ffsoa"
    fb.write_soa(p, c)
    back = fb.read_soa_host(p)
    assert list(back) == list(c)
    for k in c:
        assert back[k].tobytes() == c[k].tobytes()


def test_layout_is_aligned(tmp_path):
    n = 1000
    p = tmp_path / "d.ffsoa"
    c = cols(n)
    fb.write_soa(p, c)
    raw = open(p, "rb").read()
    assert raw[:8] == b"FFSOA01\0"
    ncols, hbytes, nrows = struct.unpack_from("<IIQ", raw, 8)
    assert (ncols, nrows) == (3, n) and hbytes % 4096 == 0
    stride = -(-n * 8 // 4096) * 4096
    assert len(raw) == hbytes + 3 * stride
    for i, k in enumerate(c):  # each column starts 4 KiB-aligned, native fp64
        assert np.frombuffer(raw, np.float64, n, hbytes + i * stride).tobytes() == c[k].tobytes()


def test_corruption_and_truncation_are_data_errors(tmp_path):
    p = tmp_path / "d.ffsoa"
    fb.write_soa(p, cols(5000))
    raw = bytearray(open(p, "rb").read())
    hbytes = struct.unpack_from("<I", raw, 12)[0]
    bad = bytearray(raw)
    bad[hbytes + 8 * 17] ^= 0x01  # flip one bit of column 0
    q = tmp_path / "bad.ffsoa"
    open(q, "wb").write(bad)
    with pytest.raises(fb.FfitError) as e:
        fb.read_soa_host(q)
    assert e.value.code == 2 and "checksum mismatch in column 'x'" in str(e.value)
    open(q, "wb").write(raw[:-100])
    with pytest.raises(fb.FfitError) as e:
        fb.read_soa_host(q)
    assert e.value.code == 2 and "truncated" in str(e.value)
    open(q, "wb").write(b"NOTSOA" + raw[6:])
    with pytest.raises(fb.FfitError) as e:
        fb.read_soa_host(q)
    assert e.value.code == 2 and "bad magic" in str(e.value)
    with pytest.raises(fb.FfitError) as e:
        fb.read_soa_host(tmp_path / "missing.ffsoa")
    assert e.value.code == 2


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 7, 100_003, 9_000_001])
def test_device_load_round_trip_and_nll(tmp_path, n):
    """Load through the pinned double-buffered upload (several 64 MiB chunks at 9e6 rows x 2
    columns), download bitwise, and the likelihood on it equals the likelihood on an
    ordinary upload."""
    rng = np.random.default_rng(n)
    c = {"x": rng.uniform(-4, 4, n), "w": rng.normal(size=n)}
    p = tmp_path / "d.ffsoa"
    fb.write_soa(p, c)
    ds, sec = fb.DataSet.load_soa(p)
    assert ds.n_rows == n and sec >= 0
    for k in c:
        assert ds.column(k).tobytes() == c[k].tobytes()
    if n:
        m = fb.Model.from_string("observable x -4 4\nparameter mu 0.1 -1 1\nparameter s 1.3 0.1 3\n"
                                 "pdf g Gaussian(x, mu, s)\n")
        assert fb.nll(m, ds).value == fb.nll(m, fb.DataSet.from_columns({"x": c["x"]})).value
    q = tmp_path / "e.ffsoa"
    ds.save_soa(q)
    assert open(q, "rb").read() == open(p, "rb").read()


@pytest.mark.gpu
def test_device_load_detects_corruption(tmp_path):
    p = tmp_path / "d.ffsoa"
    fb.write_soa(p, {"x": np.linspace(0, 1, 300_000)})
    raw = bytearray(open(p, "rb").read())
    raw[-4096 - 8] ^= 0x40
    open(p, "wb").write(raw)
    with pytest.raises(fb.FfitError) as e:
        fb.DataSet.load_soa(p)
    assert e.value.code == 2 and "checksum" in str(e.value)


def test_make_inputs_manifest(tmp_path):
    """tools/make_inputs.py: the generator's columns on disk with seed, N and sha256."""
    import hashlib
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([sys.executable, os.path.join(root, "tools", "make_inputs.py"), "--workload", "c2",
                    "--events", "20000", "--out", str(tmp_path)], check=True, capture_output=True)
    man = json.load(open(tmp_path / "c2_gauss_argus_1e7.json"))
    raw = open(tmp_path / man["file"], "rb").read()
    assert hashlib.sha256(raw).hexdigest() == man["sha256"]
    from paper_2003_12875_b200 import configs
    want, _ = fb.sample_host(fb.Model.from_string(configs.C2.text), 20000, configs.C2.data_seed)
    got = fb.read_soa_host(tmp_path / man["file"])
    assert man["seed"] == configs.C2.data_seed and man["n"] == 20000
    assert got["x"].tobytes() == want["x"].tobytes()
