"""Pin the CPU oracle against the reference's golden vectors (CPU only)."""

import numpy as np
import pytest

from conftest import load_npz
from oracle import codec as oc
from oracle import rng as orng


def test_derive_key_matches_reference(stream_golden):
    meta, _ = stream_golden
    for ent in meta.values():
        assert list(orng.derive_key(tuple(ent["parts"]))) == ent["key"]


def test_restated_philox_matches_reference_streams(stream_golden):
    meta, arr = stream_golden
    for i, ent in meta.items():
        key = ent["key"]
        ref = arr[f"u{i}"]
        for start in (0, 1, 2, 3, 5, 4000):
            got = orng.uniforms_restated(key, start, len(ref) - start)
            np.testing.assert_array_equal(got, ref[start:])
        np.testing.assert_array_equal(orng.uniforms_restated(key, 1_000_001, 37),
                                      arr[f"far{i}"])


def test_oracle_stream_class_matches(stream_golden):
    meta, arr = stream_golden
    ent = meta["3"]
    st = orng.Stream(*ent["parts"])
    a = st.uniforms(100)
    b = st.uniforms(3999)
    np.testing.assert_array_equal(np.concatenate([a, b]), arr["u3"][:4099])


def test_codec_cases_bit_exact(codec_golden):
    meta, arr = codec_golden
    for m in meta:
        ci, b, rows, d = m["case"], m["bits"], m["rows"], m["d"]
        x = arr[f"x{ci}"].astype(np.float64)
        st = orng.Stream(*m["key"])
        u = st.uniforms(rows * d) if b != 32 else None
        rmin, rscale, codes = oc.quantize(x, b, u)
        if b == 32:
            assert arr[f"wire{ci}"].tobytes() == x.tobytes()
            continue
        assert oc.wire_block(rmin, rscale, codes, b, rows, d) == arr[f"wire{ci}"].tobytes(), m
        np.testing.assert_array_equal(oc.dequantize(rmin, rscale, codes, b), arr[f"deq{ci}"])
        pb, pr, pd, pmin, pscale, pcodes = oc.parse_wire_block(arr[f"wire{ci}"].tobytes())
        assert (pb, pr, pd) == (b, rows, d)
        np.testing.assert_array_equal(pcodes, codes)


def test_multi_peer_stream_continuity():
    arr = load_npz("multi_peer.npz")
    st = orng.Stream(5, 1, 2, 3, "backward")
    for peer in (0, 2, 3):
        x = arr[f"x{peer}"].astype(np.float64)
        if x.shape[0] == 0:
            continue  # empty peers are skipped and consume no uniforms
        rmin, rscale, codes = oc.quantize(x, 1, st.uniforms(x.size))
        assert oc.wire_block(rmin, rscale, codes, 1, *x.shape) == arr[f"wire{peer}"].tobytes()


def test_known_answer_bit_layouts():
    # reference tests/test_codec.py:36-45
    assert oc.pack(np.array([[1, 0, 1, 1]]), 1) == b"\x0d"
    assert oc.pack(np.array([[3, 0, 1, 2]]), 2) == b"\x93"
    assert oc.pack(np.array([[1, 1, 1], [0, 0, 1]]), 1) == b"\x07\x04"


@pytest.mark.parametrize("b", [1, 2, 3, 4, 5, 6, 7, 8, 16])
def test_pack_roundtrip(b):
    codes = np.random.default_rng(b).integers(0, 1 << b, size=(5, 33))
    assert len(oc.pack(codes, b)) == 5 * oc.row_bytes(33, b)
    np.testing.assert_array_equal(oc.unpack(oc.pack(codes, b), 5, 33, b), codes)


def test_non_finite_rejected():
    with pytest.raises(oc.OracleCodecError):
        oc.quantize(np.array([[1.0, np.nan]]), 1, np.zeros(2))
