"""CBDICT01 / CBMEAS01 / EPI-pattern containers, byte-compatible with the reference.

The fixtures in tests/golden/ were written by the reference's own savers
(``tests/golden/make_golden.py containers``).
"""

import os

import numpy as np
import pytest

from paper_1810_01967_b200 import containers as ct

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_dictionary_reads_reference_file_and_writes_identical_bytes(tmp_path):
    d = ct.load_dictionary(os.path.join(GOLD, "small.cbdict"))
    assert d.atoms.shape == (d.d, 12) and d.lookup_table.shape == (d.d, 3)
    np.testing.assert_allclose(np.linalg.norm(d.atoms, axis=1), 1.0, rtol=1e-12)
    out = tmp_path / "copy.cbdict"
    ct.save_dictionary(d, out)
    assert out.read_bytes() == open(os.path.join(GOLD, "small.cbdict"), "rb").read()


def test_measurements_and_pattern_round_trip(tmp_path):
    Y = ct.load_measurements(os.path.join(GOLD, "small.cbmeas"))
    assert Y.shape == (24, 12) and Y.dtype == np.complex128
    out = tmp_path / "copy.cbmeas"
    ct.save_measurements(Y, out)
    assert out.read_bytes() == open(os.path.join(GOLD, "small.cbmeas"), "rb").read()
    P = ct.load_pattern(os.path.join(GOLD, "epi.json"))
    assert P.indices.shape == (12, 16) and P.lines_per_frame == 2
    ct.save_pattern(P, tmp_path / "p.json")
    assert ct.load_pattern(tmp_path / "p.json").indices.tolist() == P.indices.tolist()


def test_container_errors_match_reference(tmp_path):
    bad = tmp_path / "bad"
    bad.write_bytes(b"NOTMAGIC" + b"\0" * 64)
    with pytest.raises(ValueError, match="not a dictionary file"):
        ct.load_dictionary(bad)
    with pytest.raises(ValueError, match="not a measurement file"):
        ct.load_measurements(bad)
    blob = open(os.path.join(GOLD, "small.cbdict"), "rb").read()
    (tmp_path / "t.cbdict").write_bytes(blob[:-8])
    with pytest.raises(ValueError, match="truncated dictionary file"):
        ct.load_dictionary(tmp_path / "t.cbdict")
    (tmp_path / "h.cbdict").write_bytes(blob[:12])
    with pytest.raises(ValueError, match="truncated dictionary file"):
        ct.load_dictionary(tmp_path / "h.cbdict")
    mb = open(os.path.join(GOLD, "small.cbmeas"), "rb").read()
    (tmp_path / "t.cbmeas").write_bytes(mb[:-1])
    with pytest.raises(ValueError, match="truncated measurement file"):
        ct.load_measurements(tmp_path / "t.cbmeas")
    (tmp_path / "p.json").write_text('{"h": 8, "w": 8, "L": 2, "lines_per_frame": 2, '
                                     '"offset_rule": "random"}')
    with pytest.raises(ValueError, match="unknown offset rule"):
        ct.load_pattern(tmp_path / "p.json")


@pytest.mark.gpu
def test_device_loaders_match_host_loaders(tmp_path, monkeypatch):
    import torch
    monkeypatch.setattr(ct, "_STAGE_BYTES", 4096)        # many staging rounds on a small file
    atoms, meta = ct.load_dictionary_device(os.path.join(GOLD, "small.cbdict"))
    host = ct.load_dictionary(os.path.join(GOLD, "small.cbdict"))
    assert atoms.is_cuda and atoms.dtype == torch.complex128
    np.testing.assert_array_equal(atoms.cpu().numpy(), host.atoms)
    np.testing.assert_array_equal(meta.lookup_table, host.lookup_table)
    Yfm = ct.load_measurements_device(os.path.join(GOLD, "small.cbmeas"))
    Y = ct.load_measurements(os.path.join(GOLD, "small.cbmeas"))
    assert tuple(Yfm.shape) == (12, 24) and Yfm.dtype == torch.complex64
    np.testing.assert_array_equal(Yfm.cpu().numpy(), Y.T.astype(np.complex64))
    # a large dictionary streams through the pinned double buffer
    rng = np.random.default_rng(3)
    big = ct.Dictionary(atoms=rng.standard_normal((3000, 50)) + 1j * rng.standard_normal((3000, 50)),
                        norms=np.ones(3000), lookup_table=rng.random((3000, 3)), tr_ms=10.0, L=50)
    ct.save_dictionary(big, tmp_path / "big.cbdict")
    a2, _ = ct.load_dictionary_device(tmp_path / "big.cbdict")
    np.testing.assert_array_equal(a2.cpu().numpy(), big.atoms)
