"""TTLAB1 files straight to / from device memory (serialize.hpp:61-121)."""
import numpy as np
import pytest

from oracle import ttlab_oracle as O
from paper_2601_16734_b200 import inputs as I

pytestmark = pytest.mark.gpu


def T():
    from paper_2601_16734_b200 import ttlab
    return ttlab


def test_mps_round_trip_bit_exact(tmp_path):
    """test_core.cpp:229-241 through the device."""
    t = T()
    state = O.random_uniform_mps(5, 2, 4, 123)
    state.error = 0.125
    f = tmp_path / "v.ttlab"
    f.write_bytes(O.dumps_mps(state))
    d = t.load_mps(f)
    assert d.error() == 0.125
    assert d.info()["dtype"] == 1  # complex data stays complex128
    for a, b in zip(d.to_tensors(), state.tensors):
        assert a.shape == b.shape and a.tobytes() == b.tobytes()
    g = tmp_path / "w.ttlab"
    t.save_mps(g, d)
    assert g.read_bytes() == f.read_bytes()


def test_real_data_demoted_and_promoted_back(tmp_path):
    t = T()
    ts = I.random_mps(9, 2, 12, 4)
    state = O.MPS([x.astype(np.complex128) for x in ts], 0.5)
    f = tmp_path / "r.ttlab"
    f.write_bytes(O.dumps_mps(state))
    d = t.load_mps(f)
    assert d.info()["dtype"] == 0  # float64 on the device
    for a, b in zip(d.to_tensors(), ts):
        assert a.dtype == np.float64 and np.array_equal(a, b)
    keep = t.load_mps(f, real_if_possible=False)
    assert keep.info()["dtype"] == 1
    g = tmp_path / "r2.ttlab"
    t.save_mps(g, d)  # float64 -> complex128 with zero imaginary parts
    assert g.read_bytes() == f.read_bytes()


def test_batch_chain_save_and_large_file(tmp_path):
    """A file larger than the 32 MB staging buffers, and one chain of a batch."""
    t = T()
    big = I.random_mps(24, 2, 512, 9, complex_=True)
    f = tmp_path / "big.ttlab"
    f.write_bytes(O.dumps_mps(O.MPS(big, 0.0)))
    assert f.stat().st_size > 40 << 20  # spans several 32 MB staging chunks
    d = t.load_mps(f)
    for a, b in zip(d.to_tensors(), big):
        assert np.array_equal(a, b)
    g = tmp_path / "big2.ttlab"
    t.save_mps(g, d)
    assert g.read_bytes() == f.read_bytes()
    chains = [I.random_mps(8, 2, 8, s) for s in range(3)]
    b = t.DeviceMPS.from_batch(chains, errors=[0.0, 0.25, 0.0])
    h = tmp_path / "c1.ttlab"
    t.save_mps(h, b, chain=1)
    back = O.loads_mps(h.read_bytes())
    assert back.error == 0.25
    assert all(np.array_equal(x.real, y) and not x.imag.any() for x, y in zip(back.tensors, chains[1]))


def test_mpo_round_trip_and_use(tmp_path):
    t = T()
    W = I.laplacian_mpo(10)
    f = tmp_path / "w.ttlab"
    f.write_bytes(O.dumps_mpo(O.MPO([w.astype(np.complex128) for w in W])))
    dw = t.load_mpo(f)
    g = tmp_path / "w2.ttlab"
    t.save_mpo(g, dw)
    assert g.read_bytes() == f.read_bytes()
    psi = I.random_mps(10, 2, 8, 3)
    a = t.apply_raw(dw, psi).to_tensors()
    b = t.apply_raw(W, psi).to_tensors()
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_container_errors(tmp_path):
    """test_core.cpp:252-255 plus truncated / wrong-rank / inconsistent files."""
    t = T()
    bad = tmp_path / "bad"
    bad.write_bytes(b"garbage")
    with pytest.raises(t.NumericError):
        t.load_mps(bad)
    with pytest.raises(t.NumericError):
        t.load_mps(tmp_path / "missing")
    blob = O.dumps_mps(O.random_uniform_mps(4, 2, 3, 1))
    (tmp_path / "trunc").write_bytes(blob[:-20])
    with pytest.raises(t.NumericError):
        t.load_mps(tmp_path / "trunc")
    (tmp_path / "op").write_bytes(O.dumps_mpo(O.mpo_identity(3, 2)))
    with pytest.raises(t.NumericError):
        t.load_mps(tmp_path / "op")
    with pytest.raises(t.NumericError):
        t.load_mpo(bad)
    # bond mismatch between neighbouring tensors -> shape_error (mps.hpp:134-136)
    a = O.random_uniform_mps(4, 2, 3, 1)
    blob = bytearray(O.dumps_mps(a))
    import struct
    off = 7 + 8 + 1 + 8 + 8  # right dim of tensor 0
    blob[off:off + 8] = struct.pack("<Q", 1)  # 1 x 2 x 1 claims fewer elements than follow
    (tmp_path / "mis").write_bytes(bytes(blob))
    with pytest.raises((t.ShapeError, t.NumericError)):
        t.load_mps(tmp_path / "mis")


@pytest.mark.gpu
def test_batch_upload_download_staged():
    """Batched upload/download through the pinned staging buffers (ttg_mps_upload with count > 1,
    ttg_mps_download_batch): ragged bonds per chain (padding in the device layout), more chains
    than one staging chunk holds, bit-exact round trip, same as the per-chain download."""
    t = T()
    chains = [I.random_mps(12, 2, 8 + (c % 5) * 8, 900 + c) for c in range(37)]
    big = [I.random_mps(20, 2, 512, 990 + c) for c in range(12)]  # 4 MB sites: 8 per 32 MB chunk
    for batch in (chains, big):
        d = t.DeviceMPS.from_batch(batch)
        got = d.to_tensors_batch()
        assert len(got) == len(batch)
        for c, (g, ref) in enumerate(zip(got, batch)):
            assert len(g) == len(ref)
            for a, b in zip(g, ref):
                assert a.shape == b.shape and np.array_equal(a, b)
            for a, b in zip(d.to_tensors(c), g):
                assert np.array_equal(a, b)


@pytest.mark.gpu
def test_context_communicator_world_of_one():
    """ttg_comm_*: the context owns the NCCL communicator of the batched configs.  One GPU here:
    a single-rank communicator must initialise (ncclCommInitRank through the run-time binding of libnccl) and
    the all-gather must return the local rows; without a communicator the context is a world of one."""
    from paper_2601_16734_b200 import ttlab
    from paper_2601_16734_b200.batch import gather_chain_stats_ctx
    ctx = ttlab.Context(0)
    assert ctx.comm_info() == (1, 0)
    x = np.arange(12, dtype=np.float64) * 0.5
    assert np.array_equal(ctx.allgather_f64(x), x.reshape(1, -1))
    uid = ctx.comm_unique_id()
    assert len(uid) == ttlab.Context.COMM_ID_BYTES and any(uid)
    ctx.comm_init(1, 0, uid)
    assert ctx.comm_info() == (1, 0)
    assert np.array_equal(ctx.allgather_f64(x), x.reshape(1, -1))
    with pytest.raises(Exception):
        ctx.comm_init(1, 0, uid)  # already owns one
    rows = np.arange(15, dtype=np.float64).reshape(5, 3)
    assert np.array_equal(gather_chain_stats_ctx(ctx, rows, 5, 1), rows)
    ctx.comm_free()
    assert ctx.comm_info() == (1, 0)
