"""PAT1 / GGB1 containers, byte-identical to files the
reference wrote (tests/golden/make_golden.py, file_formats)."""

import numpy as np
import pytest

from paper_2412_03898_b200.core import DynamicCloud, GaussBall
from paper_2412_03898_b200.fileio import (read_cloud, read_tensor,
                                          write_cloud, write_tensor)


def _bytes(p):
    return np.frombuffer(p.read_bytes(), np.uint8)


def _dyn(golden):
    return DynamicCloud(golden["file_dyn_p0"], golden["file_dyn_a0"],
                        golden["file_dyn_mu"], golden["file_dyn_theta"],
                        golden["file_dyn_sigma"], golden["file_dyn_omega"])


def test_tensor_bytes_match_reference(tmp_path, golden):
    p = tmp_path / "t.pat"
    write_tensor(p, golden["file_tensor"])
    assert np.array_equal(_bytes(p), golden["file_pat"])
    write_tensor(p, np.float64(2.5))
    assert np.array_equal(_bytes(p), golden["file_pat0"])
    back = read_tensor(p)
    assert back.shape == (1,) and back[0] == 2.5      # ascontiguousarray: 1-d


def test_tensor_roundtrip_byte_stable(tmp_path, golden):
    import torch
    p, q = tmp_path / "a.pat", tmp_path / "b.pat"
    write_tensor(p, torch.as_tensor(golden["file_tensor"]))
    x = read_tensor(p)
    assert np.array_equal(x, golden["file_tensor"].astype(np.float32))
    write_tensor(q, x)
    assert p.read_bytes() == q.read_bytes()


def test_cloud_bytes_match_reference(tmp_path, golden):
    p = tmp_path / "c.ggb"
    write_cloud(p, _dyn(golden))
    assert np.array_equal(_bytes(p), golden["file_ggb"])
    balls = [GaussBall(0.5, 0.3, [1.0, 2.0, 3.0]),
             GaussBall(0.25, 0.7, [-1.5, 0.0, 0.125])]
    write_cloud(p, balls)
    assert np.array_equal(_bytes(p), golden["file_ggb_static"])
    c = read_cloud(p)
    assert c.n_basis == 0 and len(c.balls) == 2
    assert c.balls[1].mu.tolist() == [-1.5, 0.0, 0.125]


def test_cloud_roundtrip(tmp_path, golden):
    p, q = tmp_path / "a.ggb", tmp_path / "b.ggb"
    write_cloud(p, _dyn(golden))
    c = read_cloud(p)
    for k in ("p0", "a0", "mu", "theta", "sigma", "omega"):
        assert np.array_equal(getattr(c, k),
                              golden["file_dyn_" + k].astype(np.float32)), k
    write_cloud(q, c)
    assert p.read_bytes() == q.read_bytes()


def test_reader_validation(tmp_path, golden):
    p = tmp_path / "x"
    p.write_bytes(b"NOPE" + bytes(20))
    with pytest.raises(ValueError, match="bad magic"):
        read_tensor(p)
    with pytest.raises(ValueError, match="bad magic"):
        read_cloud(p)
    raw = bytes(golden["file_pat"])
    p.write_bytes(raw[:-4])
    with pytest.raises(ValueError, match="payload length"):
        read_tensor(p)
    p.write_bytes(raw[:4] + (2).to_bytes(4, "little") + raw[8:])
    with pytest.raises(ValueError, match="version"):
        read_tensor(p)
    p.write_bytes(raw[:8] + (2).to_bytes(4, "little") + raw[12:])
    with pytest.raises(ValueError, match="dtype"):
        read_tensor(p)
    raw = bytes(golden["file_ggb"])
    p.write_bytes(raw[:-1])
    with pytest.raises(ValueError, match="truncated"):
        read_cloud(p)
    p.write_bytes(raw[:24] + b"p0" + raw[26:])
    with pytest.raises(ValueError, match="channel order"):
        read_cloud(p)


def test_cloud_writer_rejects_unrepresentable(tmp_path):
    b = 2
    per_ch = DynamicCloud(np.ones(b), np.ones(b), np.zeros((b, 3)),
                          np.zeros((b, 5, 3)), np.ones((b, 5, 3)),
                          np.zeros((b, 5, 3)))
    with pytest.raises(ValueError, match="per-channel"):
        write_cloud(tmp_path / "x", per_ch)
    pf = DynamicCloud.static(np.ones(b), np.ones(b), np.zeros((b, 3)), 8,
                             basis="polyfourier")
    with pytest.raises(ValueError, match="poly"):
        write_cloud(tmp_path / "x", pf)
