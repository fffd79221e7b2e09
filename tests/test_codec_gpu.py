"""K1/K2 parity on the B200: bit-exact against the reference's golden vectors
and the CPU oracle (tolerance: none — payload bytes, row_min and row_scale
must be identical; dequantized values must equal f32(reference f64 value))."""

import numpy as np
import pytest

from conftest import load_npz

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def test_device_philox_matches_reference_streams(stream_golden):
    from paper_2303_01277_b200.codec import philox_uniforms
    meta, arr = stream_golden
    for i, ent in meta.items():
        ref = arr[f"u{i}"]
        for start in (0, 1, 2, 3, 7):
            got = philox_uniforms(ent["key"], start, len(ref) - start).cpu().numpy()
            np.testing.assert_array_equal(got, ref[start:])
        got = philox_uniforms(ent["key"], 1_000_001, 37).cpu().numpy()
        np.testing.assert_array_equal(got, arr[f"far{i}"])


def test_quantize_rows_bit_exact_vs_reference_golden(codec_golden):
    from paper_2303_01277_b200.codec import QuantConfig, dequantize_rows, quantize_rows
    from paper_2303_01277_b200.rngstream import RngStream
    meta, arr = codec_golden
    for m in meta:
        ci, b = m["case"], m["bits"]
        x = arr[f"x{ci}"]
        if b == 32:
            continue
        q = quantize_rows(torch.from_numpy(x).cuda(), QuantConfig(b), RngStream(*m["key"]))
        want = arr[f"wire{ci}"].tobytes()
        got = q.to_bytes()
        assert got == want, f"case {m}: first diff at byte " \
            f"{next(i for i in range(len(want)) if got[i] != want[i])}"
        deq = dequantize_rows(q)
        np.testing.assert_array_equal(deq.astype(np.float32), arr[f"deq{ci}"].astype(np.float32))


def test_passthrough_device_roundtrip(codec_golden):
    from paper_2303_01277_b200.codec import QuantConfig, dequantize_rows, quantize_rows
    meta, arr = codec_golden
    for m in meta:
        if m["bits"] != 32:
            continue
        x = arr[f"x{m['case']}"]
        q = quantize_rows(torch.from_numpy(x).cuda(), QuantConfig(32))
        np.testing.assert_array_equal(dequantize_rows(q), x.astype(np.float64))


def test_stream_continues_across_blocks():
    from paper_2303_01277_b200.codec import QuantConfig, quantize_rows
    from paper_2303_01277_b200.rngstream import RngStream
    arr = load_npz("multi_peer.npz")
    st = RngStream(5, 1, 2, 3, "backward")
    for peer in (0, 2, 3):
        x = arr[f"x{peer}"]
        if x.shape[0] == 0:
            continue
        assert quantize_rows(torch.from_numpy(x).cuda(), QuantConfig(1), st).to_bytes() == \
            arr[f"wire{peer}"].tobytes()


@pytest.mark.parametrize("d", [64, 100, 128, 300, 602, 1024, 1500])
@pytest.mark.parametrize("bits", [1, 2, 4, 8, 16])
def test_random_blocks_vs_oracle(d, bits):
    from oracle import codec as oc
    from oracle import rng as orng
    from paper_2303_01277_b200.codec import QuantConfig, quantize_rows
    from paper_2303_01277_b200.rngstream import RngStream
    rows = 512 if d <= 602 else 96
    rng = np.random.default_rng(2303 + d + bits)
    x = (rng.standard_normal((rows, d)) * rng.uniform(0.1, 5.0, (rows, 1))).astype(np.float32)
    x[::7] = np.maximum(x[::7], 0)   # ReLU-like rows
    st = RngStream(9, 2, 3, 1, "forward")
    st.take(5 * d + 2)               # non-zero, non-multiple-of-4 stream offset
    q = quantize_rows(torch.from_numpy(x).cuda(), QuantConfig(bits), st)
    ost = orng.Stream(9, 2, 3, 1, "forward")
    ost.uniforms(5 * d + 2)
    rmin, rscale, codes = oc.quantize(x.astype(np.float64), bits, ost.uniforms(rows * d))
    assert q.to_bytes() == oc.wire_block(rmin, rscale, codes, bits, rows, d)


def test_non_finite_rejected():
    from paper_2303_01277_b200.codec import CodecError, QuantConfig, quantize_rows
    from paper_2303_01277_b200.rngstream import RngStream
    with pytest.raises(CodecError):
        quantize_rows(torch.tensor([[1.0, float("nan")]]).cuda(), QuantConfig(1),
                      RngStream(1, 0, 1, 1, "forward"))
    with pytest.raises(CodecError):
        quantize_rows(torch.tensor([[1.0, float("inf")]]).cuda(), QuantConfig(1),
                      RngStream(1, 0, 1, 1, "forward"))
    with pytest.raises(CodecError):
        quantize_rows(np.ones((1, 2)), QuantConfig(1), None)


@pytest.mark.parametrize("d", [41, 256, 602])
@pytest.mark.parametrize("bits", [1, 2, 8, 16, 32])
@pytest.mark.parametrize("accumulate", [False, True])
def test_dequant_gather_multi_source_exact(d, bits, accumulate):
    """K2 over several wire blocks: destination t gets
    f32(f64(t if accumulate) + sum_k f64 dequant(src_k)) with sources summed in
    the listed (ascending-peer) order (trainer.py:208-216, codec.py:199-207)."""
    from oracle import codec as oc
    from paper_2303_01277_b200.codec import dequant_gather, segments_tensor
    rng = np.random.default_rng(d * 7 + bits)
    blocks, rows_per = [], [37, 0, 64, 5]
    for r in rows_per:
        x = (rng.standard_normal((r, d)) * rng.uniform(0.1, 4.0, (r, 1))).astype(np.float64)
        u = rng.random(r * d) if bits != 32 else None
        rmin, rscale, codes = oc.quantize(x.astype(np.float32).astype(np.float64), bits, u)
        blocks.append((oc.wire_block(rmin, rscale, codes, bits, r, d), oc.dequantize(rmin, rscale, codes, bits)))
    sizes = [(len(b) + 15) // 16 * 16 for b, _ in blocks]
    buf = np.zeros(sum(sizes), dtype=np.uint8)
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(int)
    for (b, _), o in zip(blocks, offs):
        buf[o:o + len(b)] = np.frombuffer(b, dtype=np.uint8)
    dbuf = torch.from_numpy(buf).cuda()
    segs = segments_tensor(rows_per, [(0, 0)] * 4, [0] * 4, [dbuf.data_ptr() + int(o) for o in offs], "cuda")
    recv = np.concatenate([v for _, v in blocks])            # flattened received rows (f64)
    R = recv.shape[0]
    ndst = 60
    # destinations: some get 0, 1 or several sources (ascending flat order)
    owner = rng.integers(0, ndst, R)
    order = np.lexsort((np.arange(R), owner))
    dst_rows, starts = np.unique(owner[order], return_index=True)
    src_ptr = np.append(starts, R).astype(np.int32)
    src_rows = order.astype(np.int32)
    ld = (d + 3) // 4 * 4
    init = rng.standard_normal((ndst + 3, ld)).astype(np.float32)
    dst = torch.from_numpy(init.copy()).cuda()
    dequant_gather(segs, 4, torch.from_numpy(dst_rows.astype(np.int32)).cuda(),
                   torch.from_numpy(src_ptr).cuda(), torch.from_numpy(src_rows).cuda(), d, bits, dst, accumulate)
    got = dst.cpu().numpy()
    want = init.copy()
    for i, t in enumerate(dst_rows):
        acc = init[t, :d].astype(np.float64) if accumulate else np.zeros(d)
        for k in range(src_ptr[i], src_ptr[i + 1]):
            acc = acc + recv[src_rows[k]]
        want[t, :d] = acc.astype(np.float32)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("d", [2, 3, 37])
def test_one_bit_row_maxima_vs_oracle(d):
    """1 bit at the row extremes: every row's maximum has hbar = (mx - mn) /
    f32(mx - mn) within an ulp of 1 (and rows with repeated maxima / ReLU
    zeros repeat that), the case the fp32 fast decision must hand to the exact
    path only when the uniform is within the error bound.  Many short rows,
    wire bytes must equal the oracle's."""
    from oracle import codec as oc
    from oracle import rng as orng
    from paper_2303_01277_b200.codec import QuantConfig, quantize_rows
    from paper_2303_01277_b200.rngstream import RngStream
    rows = 120_000 // d
    rng = np.random.default_rng(77 + d)
    x = (rng.standard_normal((rows, d)) * rng.uniform(1e-3, 1e3, (rows, 1))).astype(np.float32)
    x[::5] = np.maximum(x[::5], 0)                       # ties at the minimum
    x[1::5, : max(1, d // 2)] = x[1::5].max(axis=1, keepdims=True)   # repeated maxima
    st = RngStream(3, 1, 4, 2, "backward")
    q = quantize_rows(torch.from_numpy(x).cuda(), QuantConfig(1), st)
    ost = orng.Stream(3, 1, 4, 2, "backward")
    rmin, rscale, codes = oc.quantize(x.astype(np.float64), 1, ost.uniforms(rows * d))
    assert q.to_bytes() == oc.wire_block(rmin, rscale, codes, 1, rows, d)
