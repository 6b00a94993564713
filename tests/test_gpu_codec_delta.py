"""Codec and delta algebra on the GPU vs the oracle: bit-exact bytes, indices
and parameter values (integer/byte work and exact fp64 mul/add)."""

import numpy as np
import pytest

from conftest import random_params
from oracle import airgs_oracle as orc

pytestmark = pytest.mark.gpu


def _delta(rng, n, width, k, scale=0.05):
    from paper_2512_20943_b200.model import DeltaTensor

    idx = np.sort(rng.choice(n, k, replace=False))
    rows = rng.normal(0, scale, (k, width))
    return DeltaTensor(n, width, {int(i): r for i, r in zip(idx, rows)}), idx, rows


@pytest.mark.parametrize("n,deg", [(5, 0), (37, 1), (1000, 0), (4097, 0)])
def test_gsai_round_trip_bit_exact(n, deg):
    from paper_2512_20943_b200 import codec
    from paper_2512_20943_b200.model import GaussianFrame

    rng = np.random.default_rng(n)
    p = random_params(rng, n, deg)
    blob = codec.encode_frame(GaussianFrame(params=p, frame_index=3, group_key=3)).to_bytes()
    assert blob == orc.gsai_encode(p, 3, 3)
    back = codec.decode_frame(codec.AttributeImageSet.from_bytes(blob))
    ref, fi, gk = orc.gsai_decode(blob)
    np.testing.assert_array_equal(back.params, ref)
    assert (back.frame_index, back.group_key) == (fi, gk) == (3, 3)


def test_gsai_constant_plane_exact():
    from paper_2512_20943_b200 import codec
    from paper_2512_20943_b200.model import GaussianFrame

    params = np.tile(np.linspace(-1, 1, 17), (5, 1))
    back = codec.decode_frame(codec.encode_frame(GaussianFrame(params=params)))
    np.testing.assert_array_equal(back.params, params)


def test_gsai_errors(rng):
    from paper_2512_20943_b200 import codec
    from paper_2512_20943_b200.errors import CapacityError, DecodeError
    from paper_2512_20943_b200.model import GaussianFrame

    f = GaussianFrame(params=random_params(rng, 10))
    with pytest.raises(CapacityError):
        codec.encode_frame(f, width=3, height=3)
    blob = bytearray(codec.encode_frame(GaussianFrame(params=random_params(rng, 4))).to_bytes())
    with pytest.raises(DecodeError):
        codec.AttributeImageSet.from_bytes(b"XXXX" + bytes(blob[4:]))
    with pytest.raises(DecodeError):
        codec.AttributeImageSet.from_bytes(bytes(blob[: len(blob) // 2]))


@pytest.mark.parametrize("n,k,step", [(12, 3, 1e-4), (5000, 1000, 1e-4), (100000, 2, 1e-3), (300, 300, 1e-2)])
def test_gsdp_round_trip_bit_exact(n, k, step):
    from paper_2512_20943_b200 import codec

    rng = np.random.default_rng(k)
    d, idx, rows = _delta(rng, n, 17, k)
    pay = codec.encode_delta(d, step, frame_index=7, base_key=2)
    ref = orc.gsdp_encode(idx, rows, step, 7, 2)
    assert pay.data == ref
    assert pay.payload_bytes == orc.gsdp_size(idx, rows, step)
    back = codec.decode_delta(pay, n, 17)
    ri, rr, *_ = orc.gsdp_decode(ref, n, 17)
    np.testing.assert_array_equal(back.indices(), ri)
    got = back.entries
    for i, r in zip(ri.tolist(), rr):
        np.testing.assert_array_equal(got[i], r)


def test_gsdp_infer_width_and_count(rng):
    from paper_2512_20943_b200 import codec

    d, idx, rows = _delta(rng, 8, 17, 1, scale=1.0)
    back = codec.decode_delta(codec.encode_delta(d, 1e-4))
    assert back.param_width == 17
    assert back.base_count == int(idx[-1]) + 1


def test_gsdp_empty_and_subquantum():
    from paper_2512_20943_b200 import codec
    from paper_2512_20943_b200.model import DeltaTensor

    pay = codec.encode_delta(DeltaTensor.empty(10, 17), 1e-4)
    assert pay.payload_bytes == codec.DELTA_HEADER_BYTES and pay.entry_count == 0
    assert codec.decode_delta(pay, 10, 17).is_empty()
    sub = DeltaTensor(4, 17, {1: np.full(17, 1e-4)})
    assert codec.encode_delta(sub, 1e-3).entry_count == 0


def test_gsdp_errors(rng):
    from paper_2512_20943_b200 import codec
    from paper_2512_20943_b200.errors import DecodeError, StructuralError
    from paper_2512_20943_b200.model import DeltaTensor

    pay = codec.encode_delta(DeltaTensor(4, 17, {0: np.ones(17)}), 1e-3)
    with pytest.raises(DecodeError):
        codec.decode_delta(b"XXXX" + pay.data[4:], 4, 17)
    with pytest.raises(DecodeError):
        codec.decode_delta(pay.data[:-8], 4, 17)
    with pytest.raises(DecodeError):
        codec.decode_delta(pay.data[:10], 4, 17)
    # 11-byte varint -> "varint too long" (reference order)
    import struct

    bad = struct.pack("<4sIIId", b"GSDP", 0, 0, 1, 1e-3) + bytes([0xFF] * 10 + [0x01]) + bytes(68)
    with pytest.raises(DecodeError, match="too long"):
        codec.decode_delta(bad, 4, 17)
    with pytest.raises(StructuralError):
        codec.decode_delta(codec.encode_delta(DeltaTensor(100, 17, {99: np.ones(17)}), 1e-3), 50, 17)
    with pytest.raises(StructuralError):
        codec.encode_delta(DeltaTensor.empty(4, 17), 0.0)


def test_gsdp_duplicate_index_last_wins():
    """A zero gap repeats an index; the dict keeps the last row
    (ss/codec.py:247)."""
    import struct

    from paper_2512_20943_b200 import codec

    q = np.arange(34, dtype="<i4").reshape(2, 17)
    blob = struct.pack("<4sIIId", b"GSDP", 0, 0, 2, 0.5) + bytes([3, 0]) + q.tobytes()
    back = codec.decode_delta(blob, 6, 17)
    ri, rr, *_ = orc.gsdp_decode(blob, 6, 17)
    assert list(back.entries) == [3] == ri.tolist()
    np.testing.assert_array_equal(back.entries[3], rr[0])


def test_compose_apply_bit_exact(rng):
    from paper_2512_20943_b200.model import CanonicalSpace, GaussianFrame, apply_delta, compose_deltas

    n = 3000
    a, ai, ar = _delta(rng, n, 17, 600)
    b, bi, br = _delta(rng, n, 17, 900)
    # make some sums cancel below eps
    c = compose_deltas([a, b.negate(), a])
    ref_i, ref_r = orc.compose([(ai, ar), (bi, -br), (ai, ar)])
    np.testing.assert_array_equal(c.indices(), ref_i)
    got = c.entries
    for i, r in zip(ref_i.tolist(), ref_r):
        np.testing.assert_array_equal(got[i], r)
    canon = random_params(rng, n)
    space = CanonicalSpace(GaussianFrame(params=canon), capacity_U=n)
    fr = apply_delta(space, c, frame_index=4)
    np.testing.assert_array_equal(fr.params, orc.apply(canon, ref_i, ref_r))
    assert (fr.frame_index, fr.group_key) == (4, 0)


def test_compose_cancellation_drops_rows():
    from paper_2512_20943_b200.model import DeltaTensor, compose_deltas

    a = DeltaTensor(5, 17, {1: np.full(17, 0.5), 2: np.full(17, 1.0)})
    b = DeltaTensor(5, 17, {1: np.full(17, -0.5)})
    c = compose_deltas([a, b])
    assert sorted(c.entries) == [2]
    assert compose_deltas([]).base_count == 0


def test_diff_frames_exact(rng):
    from paper_2512_20943_b200.model import CanonicalSpace, GaussianFrame, apply_delta, diff_frames

    a = random_params(rng, 500)
    b = a.copy()
    b[::7, 0:3] += rng.normal(0, 0.01, (len(b[::7]), 3))
    d = diff_frames(GaussianFrame(params=a), GaussianFrame(params=b))
    ri, rr = orc.from_dense(b - a)
    np.testing.assert_array_equal(d.indices(), ri)
    back = apply_delta(CanonicalSpace(GaussianFrame(params=a), 500), d)
    np.testing.assert_array_equal(back.params, orc.apply(a, ri, rr))


def _fused_vs_two_step(blob, n, w=17, seed=0):
    import torch

    from paper_2512_20943_b200 import codec, device as dv
    from paper_2512_20943_b200.model import apply_overlay

    rng = np.random.default_rng(seed)
    canon = dv.upload_params(rng.normal(size=(n, w)))
    fused = codec.decode_apply_device(blob, canon, n, w)
    delta, _ = codec.decode_delta_device(blob, n, w)
    two = apply_overlay(canon, n, delta.overlay())
    assert torch.equal(fused[:, :n], two[:, :n])
    return fused


@pytest.mark.parametrize("n,k,step", [(12, 3, 1e-4), (5000, 1000, 1e-4), (300000, 60000, 1e-4), (100000, 2, 1e-3),
                                      (300, 300, 1e-2), (70000, 69999, 1e-3)])
def test_fused_decode_apply_equals_decode_then_apply(n, k, step):
    """airgs_gsdp_decode_apply (single-pass varint decode + streamed rows into
    a copy of the canonical planes) == decode_delta + apply_delta, bit for
    bit, from tiny to C2-sized payloads (60k entries), dense and sparse."""
    from paper_2512_20943_b200 import codec

    rng = np.random.default_rng(k + n)
    d, idx, rows = _delta(rng, n, 17, k)
    _fused_vs_two_step(codec.encode_delta(d, step).data, n)


def test_fused_decode_apply_edge_cases_and_errors():
    """Empty delta (params = canonical), a duplicate index (the exact path's
    dict semantics), and every malformed payload raising the reference's
    error class through the fused entry, in checked and deferred mode."""
    import ctypes
    import struct

    from paper_2512_20943_b200 import _lib, codec, device as dv
    from paper_2512_20943_b200.errors import DecodeError, StructuralError
    from paper_2512_20943_b200.model import DeltaTensor

    _fused_vs_two_step(codec.encode_delta(DeltaTensor.empty(10, 17), 1e-4).data, 10)
    q = np.arange(34, dtype="<i4").reshape(2, 17)
    _fused_vs_two_step(struct.pack("<4sIIId", b"GSDP", 0, 0, 2, 0.5) + bytes([3, 0]) + q.tobytes(), 6)
    canon = dv.upload_params(np.zeros((4, 17)))
    pay = codec.encode_delta(DeltaTensor(4, 17, {0: np.ones(17)}), 1e-3)
    bad = [(pay.data[:-8], DecodeError), (pay.data[:10], DecodeError),
           (struct.pack("<4sIIId", b"GSDP", 0, 0, 1, 1e-3) + bytes([0xFF] * 10 + [0x01]) + bytes(68), DecodeError),
           (codec.encode_delta(DeltaTensor(100, 17, {99: np.ones(17)}), 1e-3).data, StructuralError)]
    for blob, exc in bad:
        with pytest.raises(exc):
            codec.decode_apply_device(blob, canon, 4, 17)
    eng = _lib.engine()
    flags = ctypes.c_uint32(0)
    for blob, _ in bad:
        if len(blob) < codec.DELTA_HEADER_BYTES:
            continue  # header errors are raised by the host-side header parse, deferred or not
        eng.call("airgs_defer", 1, ctypes.byref(flags))
        try:
            codec.decode_apply_device(blob, canon, 4, 17)
        finally:
            eng.call("airgs_defer", 0, ctypes.byref(flags))
        assert flags.value != 0  # folded into the deferred word, no exception


@pytest.mark.gpu
def test_decode_apply_ahead_sequence_equals_one_call_path():
    """airgs_gsdp_decode_apply_ahead under deferred checking (the pipelined
    probe): each frame's varint scan runs ahead on the side stream while the
    previous frame is applied; a frame decoded out of order (no matching
    prescan), a repeated payload and the last frame (no next) all give
    params bit-identical to the one-call path, and a malformed next payload
    (scanned ahead) or frame folds into the deferred word."""
    import ctypes
    import struct

    import torch

    from paper_2512_20943_b200 import _lib, codec, device as dv

    n, w = 20000, 17
    rng = np.random.default_rng(7)
    canon = dv.upload_params(rng.normal(size=(n, w)))
    blobs = []
    for k in (4000, 1, 9000, 2500, 4000):
        d, _, _ = _delta(rng, n, w, k)
        blobs.append(codec.encode_delta(d, 1e-4).data)
    devs = [torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda() for b in blobs]
    want = [codec.decode_apply_device(b, canon, n, w, payload_dev=p) for b, p in zip(blobs, devs)]
    bad = struct.pack("<4sIIId", b"GSDP", 0, 0, 1, 1e-3) + bytes([0xFF] * 10 + [0x01]) + bytes(68)
    bad_dev = torch.frombuffer(bytearray(bad), dtype=torch.uint8).cuda()
    # call order: 0,1,2 in sequence, 4 out of order (prescan of 3 unused), 3, 3 again, last without next
    order = [(0, 1), (1, 2), (2, 3), (4, 3), (3, 3), (3, None), (0, None)]
    eng = _lib.engine()
    flags = ctypes.c_uint32(0)
    got = []
    eng.call("airgs_defer", 1, ctypes.byref(flags))
    try:
        for t, nxt in order:
            ahead = None if nxt is None else (blobs[nxt], devs[nxt])
            got.append((t, codec.decode_apply_device(blobs[t], canon, n, w, payload_dev=devs[t], ahead=ahead)))
    finally:
        eng.call("airgs_defer", 0, ctypes.byref(flags))
    assert flags.value == 0
    for t, out in got:
        assert torch.equal(out[:, :n], want[t][:, :n]), t
    # a malformed frame inside the pipelined sequence folds into the deferred word
    eng.call("airgs_defer", 1, ctypes.byref(flags))
    try:
        codec.decode_apply_device(blobs[0], canon, n, w, payload_dev=devs[0], ahead=(bad, bad_dev))
        codec.decode_apply_device(bad, canon, n, w, payload_dev=bad_dev, ahead=None)
    finally:
        eng.call("airgs_defer", 0, ctypes.byref(flags))
    assert flags.value != 0
