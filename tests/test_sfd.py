"""SFD1 / SWB1 containers (sfd.hpp; acceptance.cpp:681-727): byte-identical files to the
reference writers, reference files read back exactly, the reference reader accepts ours,
and the reader's error codes.  CPU (no GPU needed)."""
import os

import numpy as np
import pytest

import oracle
from paper_2507_12144_b200 import sfd
import paper_2507_12144_b200 as S

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="needs oracle/_ref (reference build)")


def test_sfd_bytes_identical_and_roundtrip(tmp_path):
    x = oracle.random_field((3, 9, 16), 70)
    ref_path, our_path = tmp_path / "ref.sfd", tmp_path / "ours.sfd"
    oracle.ref().write_sfd(ref_path, 0, x)
    sfd.write_sfd(our_path, S.SphericalField(S.build_equiangular(9, 16), x))
    assert ref_path.read_bytes() == our_path.read_bytes()
    got = sfd.read_sfd(ref_path)
    assert got.channel_names == ["ch0", "ch1", "ch2"]
    assert np.array_equal(got.field.data, x)  # bit-exact fp64
    code, back = oracle.ref().read_sfd(our_path)
    assert code == 0 and np.array_equal(back, x)


def test_weights_bytes_identical_and_roundtrip(tmp_path):
    w1 = oracle.random_field((4, 3, 1), 71)[..., 0]
    b1 = oracle.random_field((4, 1, 1), 72)[:, 0, 0]
    ref_path, our_path = tmp_path / "ref.swb", tmp_path / "ours.swb"
    oracle.ref().write_weights(ref_path, w1, b1)
    sfd.write_weights(our_path, [sfd.NamedTensor("w1", [4, 3], w1), sfd.NamedTensor("b1", [4], b1)],
                      {"model": "fcn3", "version": 3})
    assert ref_path.read_bytes() == our_path.read_bytes()
    got = sfd.read_weights(ref_path)
    assert [t.name for t in got.tensors] == ["w1", "b1"] and got.meta == {"model": "fcn3", "version": 3}
    assert np.array_equal(got.tensors[0].data, w1) and np.array_equal(got.tensors[1].data, b1)


def test_reader_error_codes_match_reference(tmp_path):
    x = oracle.random_field((1, 4, 8), 73)
    good = tmp_path / "g.sfd"
    sfd.write_sfd(good, S.SphericalField(S.build_gaussian(4, 8), x))
    raw = good.read_bytes()
    cases = {
        "bad_magic": b"XFD1" + raw[4:],
        "payload_length_mismatch": raw[:-8],
        "unknown_grid_kind": raw.replace(b'"gaussian"', b'"hexagonl"'),
        "header_mismatch": raw[:4] + (10 ** 6).to_bytes(4, "little") + raw[8:],
    }
    for want, data in cases.items():
        p = tmp_path / f"{want}.sfd"
        p.write_bytes(data)
        with pytest.raises(sfd.IoError) as ei:
            sfd.read_sfd(p)
        assert ei.value.code == getattr(sfd.IoErrorCode, want)
        code, _ = oracle.ref().read_sfd(p)
        assert code == 1 + int(getattr(sfd.IoErrorCode, want)), want  # same verdict as the reference
