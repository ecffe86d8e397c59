"""CPU tests of the product's host logic: exact parameter derivation, file
formats, containers, validation errors, the C ABI's host-side RNG, DDP
sharding (gloo, world size 2).  No kernel launches."""

import os
import socket
import tempfile

import numpy as np
import pytest

import paper_2207_14696_b200 as fg
from paper_2207_14696_b200 import _native as N
from paper_2207_14696_b200 import ddp, formats
from paper_2207_14696_b200.sampler import rng_block_from_numpy, rng_block_to_numpy
from paper_2207_14696_b200.vq import VqParams, _fit_from_sample
from paper_2207_14696_b200.sq import sq_decode_table, sq_thresholds, _quantile_lerp, \
    _order_stat_ranks
from oracle import codecs as oc


# ------------------------------------------------------------------- ABI

def _declared_symbols():
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "featgrind_b200.h")).read()
    import re
    return sorted(set(re.findall(r"^(?:int|int64_t|const char\*)\s+\*?(fg_[a-z0-9_]+)\(", hdr,
                                 re.M)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = N.lib()
    declared = _declared_symbols()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(N.exported_symbols())
    assert lib.fg_version() == 100


def test_abi_argument_errors_without_gpu():
    # argument validation happens before any CUDA call and maps to FG_EUSAGE
    rc = N.lib().fg_sample_layer(None, None, 10, None, None, 4, 0, None, None, None, 10, None,
                                 None, None, 0, None, None)
    assert rc == N.FG_EUSAGE
    assert b"fanout" in N.lib().fg_last_error()
    with pytest.raises(fg.DataError):
        N.call("fg_sq_encode", None, 0, 4, 4, 9, None, None, None, 16, None)


# ------------------------------------------------------------------- SQ

def test_thresholds_and_lut_reproduce_reference_codes(sq_golden):
    z = sq_golden
    for key in [k for k in z.files if k.endswith("/emin_emax") and "/k" in k]:
        name, kk = key.split("/")[:2]
        k = int(kk[1:])
        x = z[f"{name}/x"]
        p = fg.SqParams(k, *map(float, z[key]))
        thr = sq_thresholds(p, 32)
        half = 1 << (k - 1)
        off = np.searchsorted(thr, np.abs(x), side="right")
        codes = (x >= 0).astype(np.int64) if k == 1 else np.where(x >= 0, half + off,
                                                                    half - 1 - off)
        ref = oc.row_codes(z[f"{name}/k{k}/payload"].tobytes(), x.shape[1], k,
                           np.arange(x.shape[0]))
        assert np.array_equal(codes, ref), key
        assert np.array_equal(sq_decode_table(p)[ref], z[f"{name}/k{k}/decoded"]), key


def test_thresholds_are_tight():
    p = fg.SqParams(5, -3.25, 2.5)
    thr = sq_thresholds(p, 32)
    below = np.nextafter(thr, np.float32(0))
    assert (oc.sq_codes(thr, 5, p.e_min, p.e_max) - 16 == np.arange(1, 16)).all()
    assert (oc.sq_codes(below, 5, p.e_min, p.e_max) - 16 == np.arange(0, 15)).all()
    thr64 = sq_thresholds(p, 64)
    assert (oc.sq_codes(thr64, 5, p.e_min, p.e_max) - 16 == np.arange(1, 16)).all()


def test_quantile_restatement_matches_numpy():
    r = np.random.default_rng(1)
    for _ in range(200):
        m = int(r.integers(1, 3000))
        v = np.sort(np.log2(np.abs(r.standard_normal(m)) + 1e-4))
        for q in (0.005, 0.995, 0.0, 0.2, 1.0):
            a, b = _order_stat_ranks(m, q)
            assert _quantile_lerp(v[a], v[b], m, q) == np.quantile(v, q)


def test_sq_params_validation():
    with pytest.raises(fg.DataError):
        fg.SqParams(0, 0.0, 1.0)
    with pytest.raises(fg.DataError):
        fg.SqParams(3, 1.0, 1.0)
    with pytest.raises(fg.DataError):
        fg.SqParams(3, 0.0, 1.0, 0.3)
    fg.SqParams(1, 0.0, 0.0)


def test_sq_compression_ratio():
    for k, cr in [(1, 32.0), (2, 16.0), (4, 8.0), (8, 4.0)]:
        c = fg.SqCodec(fg.SqParams(k, -1.0, 1.0), 4, 8, bytes((4 * 8 * k + 7) // 8))
        assert fg.sq_compression_ratio(c)[0] == cr


def test_sqf1_bytes_and_roundtrip(sq_golden):
    z = sq_golden
    x = z["conftest/x"]
    p = fg.SqParams(3, *map(float, z["conftest/k3/emin_emax"]))
    c = fg.SqCodec(p, x.shape[0], x.shape[1], z["conftest/k3/payload"].tobytes())
    with tempfile.TemporaryDirectory() as t:
        path = os.path.join(t, "a.sqf")
        fg.save_sq(c, path)
        assert open(path, "rb").read() == z["conftest/k3/sqf1"].tobytes()
        c2 = fg.load_sq(path)
        assert c2 == c
        raw = open(path, "rb").read()
        open(path, "wb").write(raw[:-1])
        with pytest.raises(fg.FormatError):
            fg.load_sq(path)
        open(path, "wb").write(b"XQF1" + raw[4:])
        with pytest.raises(fg.FormatError):
            fg.load_sq(path)


# ------------------------------------------------------------------- VQ

def _golden_codec(z, name):
    x = z[f"{name}/x"]
    w, L, metric_id, layout_id = (int(v) for v in z[f"{name}/params"][:4])
    p = fg.VqParams(w, L, ("euclidean", "cosine")[metric_id],
                    ("packed", "byte_aligned")[layout_id])
    ent = z[f"{name}/entries"]
    flat = z[f"{name}/books"]
    books, pos = [], 0
    for pi, sl in enumerate(p.part_slices(x.shape[1])):
        cnt = int(ent[pi]) * (sl.stop - sl.start)
        books.append(flat[pos:pos + cnt].reshape(int(ent[pi]), sl.stop - sl.start))
        pos += cnt
    codes = z[f"{name}/codes"]
    return fg.VqCodec(p, x.shape[1], tuple(books), codes=codes, n=codes.shape[0])


@pytest.mark.parametrize("name", ["cos_w4_L16", "cos_narrow", "cos_zeros", "euc_w8_L256"])
def test_vqf1_bytes_and_roundtrip(vq_golden, name):
    c = _golden_codec(vq_golden, name)
    with tempfile.TemporaryDirectory() as t:
        path = os.path.join(t, "a.vqf")
        fg.save_vq(c, path)
        assert open(path, "rb").read() == vq_golden[f"{name}/vqf1"].tobytes()
        c2 = fg.load_vq(path)
        assert np.array_equal(c2.codes, c.codes)
        raw = open(path, "rb").read()
        open(path, "wb").write(raw[:-1])
        with pytest.raises(fg.FormatError):
            fg.load_vq(path)


def test_vq_compression_ratio_arithmetic():
    mk = lambda w, L, lay="packed": fg.VqCodec(  # noqa: E731
        fg.VqParams(w, L, code_layout=lay), w, (np.zeros((2, w), np.float32),))
    assert round(fg.vq_compression_ratio(mk(16, 2048)).theoretical, 1) == 46.5
    assert round(fg.vq_compression_ratio(mk(100, 16384)).theoretical, 1) == 228.6
    assert fg.vq_compression_ratio(mk(16, 2048, "byte_aligned")).realized == 32.0
    assert fg.vq_compression_ratio(mk(4, 256)).realized == 16.0


def test_vq_params_validation():
    for bad in [dict(width=0, length=4), dict(width=2, length=1), dict(width=2, length=4,
                                                                       metric="l1")]:
        with pytest.raises(fg.DataError):
            fg.VqParams(**bad)


# ------------------------------------------------------------ containers

def test_fmat_csrg_bytes(formats_golden):
    z = formats_golden
    with tempfile.TemporaryDirectory() as t:
        p = os.path.join(t, "f")
        formats.write_fmat(p, z["x"])
        assert open(p, "rb").read() == z["fmat1"].tobytes()
        assert np.array_equal(formats.read_fmat(p), z["x"])
        q = os.path.join(t, "g")
        formats.write_csrg(q, 6, z["row_offsets"], z["col_indices"], True)
        assert open(q, "rb").read() == z["csrg1"].tobytes()
        n, off, col, loops = formats.read_csrg(q)
        assert n == 6 and loops and np.array_equal(col, z["col_indices"])


def test_csr_validation(sampler_golden):
    z = sampler_golden
    g = fg.CsrGraph(2000, z["graph/pa2000/row_offsets"], z["graph/pa2000/col_indices"])
    assert g.has_self_loops and g.nnz == z["graph/pa2000/col_indices"].size
    with pytest.raises(fg.DataError):  # asymmetric
        fg.CsrGraph(3, np.array([0, 1, 1, 1]), np.array([1]))
    with pytest.raises(fg.DataError):  # unsorted row
        fg.CsrGraph(3, np.array([0, 2, 3, 4]), np.array([2, 1, 0, 0]))
    with pytest.raises(fg.DataError):  # partial self loops
        fg.CsrGraph(2, np.array([0, 1, 1]), np.array([0]))
    with pytest.raises(fg.DataError):
        fg.FeatureMatrix(np.array([[np.nan]], np.float32))


# ---------------------------------------------------------- host RNG (C)

@pytest.mark.parametrize("seed", [0, 3, 2024])
def test_c_host_permutation_matches_numpy(seed):
    rng = np.random.default_rng(seed)
    blk = rng_block_from_numpy(rng.bit_generator.state)
    inc = rng.bit_generator.state["state"]["inc"]
    ids = np.arange(5, 40005, 7, dtype=np.int64)
    ref = rng.permutation(ids)
    mine = ids.copy()
    N.call("fg_rng_permutation_host", blk.ctypes.data, mine.ctypes.data, mine.size)
    assert np.array_equal(ref, mine)
    st = rng_block_to_numpy(blk, inc)
    ref_st = rng.bit_generator.state
    assert st["state"]["state"] == ref_st["state"]["state"]
    assert st["has_uint32"] == ref_st["has_uint32"]
    if st["has_uint32"]:
        assert st["uinteger"] == ref_st["uinteger"]


# ------------------------------------------------------------------ DDP

def test_ddp_sharding_helpers():
    ids = np.array([9, 3, 3, 7, 1, 12])
    assert ddp.shard_ids(ids, 0, 2).tolist() == [1, 7, 12]
    assert ddp.shard_ids(ids, 1, 2).tolist() == [3, 9]
    assert ddp.rank_seed(0, 0, 1, 2) == 1 and ddp.rank_seed(5, 1, 0, 4) == 24


def _vq_sample():
    import torch
    return torch.randn(50, 10, generator=torch.Generator().manual_seed(0), dtype=torch.float64)


def _fake_fit(owner):
    """Stand-in for the GPU k-means (no kernels on CPU): depends on the part's
    points and its restart seeds, records which rank fitted it."""
    def fit(pts, p, capacity, seeds):
        v = float(seeds[0] % 997) + float(pts.sum())
        return np.full((2, pts.shape[1]), v, np.float32), {"owner": owner}
    return fit


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nb = ddp.agree_num_batches(10 + rank)
        flat = torch.full((5,), float(rank + 1))
        ddp.average_flat_(flat)
        mx = ddp.max_over_ranks(0.5 * (rank + 1))
        shard = ddp.shard_ids(np.arange(11), rank, world)
        # sharded preprocessing: row blocks + all-gather, round-robin VQ parts
        n, stride = 11, 3
        buf = ddp.padded_rows(n, stride, world, "cpu")
        r0, r1, _ = ddp.row_block(n, rank, world)
        buf[r0:r1] = (torch.arange(r0, r1)[:, None] * 7 + torch.arange(stride)).to(torch.uint8)
        ddp.allgather_rows_(buf, n)
        rows = buf[:n].tolist()
        c = _fit_from_sample(_vq_sample(), VqParams(3, 4, metric="euclidean"), 10, 32,
                             np.random.default_rng(5), group=dist.group.WORLD,
                             fit_part=_fake_fit(rank))
        books = [b.tolist() for b in c.codebooks]
        owners = [st["owner"] for st in c.fit_stats]
        q.put((rank, nb, flat.tolist(), mx, shard.tolist(), rows, books, owners))
    finally:
        dist.destroy_process_group()


def test_ddp_gloo_world2():
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(60)
    assert [o[1] for o in out] == [10, 10]
    assert out[0][2] == [1.5] * 5 and out[1][2] == [1.5] * 5
    assert out[0][3] == 1.0
    assert out[0][4] == [0, 2, 4, 6, 8, 10] and out[1][4] == [1, 3, 5, 7, 9]
    want = [[(r * 7 + j) for j in range(3)] for r in range(11)]
    assert out[0][5] == want and out[1][5] == want
    single = _fit_from_sample(_vq_sample(), VqParams(3, 4, metric="euclidean"), 10, 32,
                              np.random.default_rng(5), fit_part=_fake_fit(0))
    assert out[0][6] == out[1][6] == [b.tolist() for b in single.codebooks]
    assert out[0][7] == out[1][7] == [p % 2 for p in range(4)]   # parts round-robin


def test_measured_report_semantics_follow_the_reference():
    """measure.SimReport / compare_reports / render_text keep the reference's
    validation and dict form (pipeline.py:224-383)."""
    from paper_2207_14696_b200.errors import DataError
    from paper_2207_14696_b200.measure import SimReport, compare_reports, render_text
    wl = {"graph_n": 10, "num_batches": 2, "fanouts": [5], "batch_size": 4, "seed": 0,
          "measured_step_us": 1.0}
    a = SimReport("vq", 1.0, 0.1, 0.5, 2.0, 3.6, 64.0, 1.0, 100, 25.0, wl)
    b = SimReport("sq", 1.0, 0.1, 1.0, 2.0, 4.1, 64.0, 1.0, 400, 100.0,
                  dict(wl, measured_step_us=2.0))
    assert SimReport.from_dict(a.to_dict()) == a
    out = compare_reports(b, [a])
    assert out[0].speedup_vs_baseline == 1.0 and abs(out[1].speedup_vs_baseline - 4.1 / 3.6) < 1e-12
    assert "speedup" in render_text(out).splitlines()[0]
    with pytest.raises(DataError):
        SimReport("x", 1.0, 0.0, 0.0, 0.0, 2.0, 0.0, 1.0, 0, 1.0, wl)
    with pytest.raises(DataError):
        compare_reports(a, [SimReport("y", 1, 0, 0, 0, 1, 0, 1.0, 0, 1.0, dict(wl, seed=1))])
    with pytest.raises(DataError):
        SimReport.from_dict({"label": "z"})


def test_sorted_unique_ids_never_aliases_the_input():
    """The fast path (already strictly increasing ids) must copy: the sampler
    permutes the returned array in place (fg_rng_permutation_host)."""
    from paper_2207_14696_b200.graph import sorted_unique_ids
    a = np.arange(10, dtype=np.int64)
    out = sorted_unique_ids(a)
    out[:] = 0
    assert np.array_equal(a, np.arange(10))
    assert np.array_equal(sorted_unique_ids(np.array([5, 3, 3, 9])), [3, 5, 9])
