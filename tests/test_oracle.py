"""Pin the CPU oracle (oracle/) against the reference's golden vectors and
numpy itself.  CPU only."""

import numpy as np
import pytest

from oracle import codecs as oc
from oracle.pcg64 import Pcg64Stream, advance_state
from oracle.sampler import sample_batches_oracle


# ---------------------------------------------------------------- PCG64

@pytest.mark.parametrize("seed", [0, 1, 7, 12345])
def test_pcg_permutation_and_choice_match_numpy(seed):
    rng = np.random.default_rng(seed)
    s = Pcg64Stream.from_numpy(rng.bit_generator.state)
    ids = np.arange(0, 3000, 3)
    assert np.array_equal(rng.permutation(ids), s.permute(ids))
    r = np.random.default_rng(seed + 99)
    for _ in range(60):
        pop = int(r.integers(2, 800))
        f = int(r.integers(1, pop))
        assert list(rng.choice(pop, f, replace=False)) == s.choice_noreplace(pop, f)
    st = rng.bit_generator.state
    assert st["state"]["state"] == s.state
    assert st["has_uint32"] == s.has32
    if s.has32:
        assert st["uinteger"] == s.buf


def test_pcg_fisher_yates_branch():
    # pop > 10000 and f > pop // 50 -> numpy's partial Fisher-Yates branch
    rng = np.random.default_rng(5)
    s = Pcg64Stream.from_numpy(rng.bit_generator.state)
    for pop, f in [(12000, 300), (20001, 500), (10001, 9000)]:
        assert list(rng.choice(pop, f, replace=False)) == s.choice_noreplace(pop, f)
    assert rng.bit_generator.state["state"]["state"] == s.state


def test_pcg_advance():
    s = Pcg64Stream.seeded(3)
    st0 = s.state
    for _ in range(1000):
        s.next64()
    assert advance_state(st0, s.inc, 1000) == s.state


# ------------------------------------------------------------------- SQ

def test_sq_oracle_matches_reference_golden(sq_golden):
    z = sq_golden
    for key in [k for k in z.files if k.endswith("/emin_emax") and "/k" in k]:
        name, kk = key.split("/")[:2]
        k = int(kk[1:])
        x = z[f"{name}/x"]
        e_min, e_max = oc.sq_fit(x, k)
        assert (e_min, e_max) == tuple(z[key]), key
        codes = oc.sq_codes(x, k, e_min, e_max)
        assert oc.pack_msb(codes, k) == z[f"{name}/k{k}/payload"].tobytes(), key
        dec = oc.sq_dequant_rows(z[f"{name}/k{k}/payload"].tobytes(), x.shape[0], x.shape[1],
                                 k, e_min, e_max)
        assert np.array_equal(dec, z[f"{name}/k{k}/decoded"]), key
        rows = z[f"{name}/k{k}/rows"]
        g = oc.sq_dequant_rows(z[f"{name}/k{k}/payload"].tobytes(), x.shape[0], x.shape[1], k,
                               e_min, e_max, rows)
        assert np.array_equal(g, z[f"{name}/k{k}/gathered"]), key


def test_sq_frozen_reference_values(sq_golden):
    # test_sq.py:71-75: codes [6,0,4,4,7,0,4,3,7] at k=3 over [-4, 0]
    x = sq_golden["specials/x"]
    codes = oc.sq_codes(x, 3, -4.0, 0.0)
    assert codes.reshape(-1).tolist() == [6, 0, 4, 4, 7, 0, 4, 3, 7]
    assert oc.pack_msb(codes, 3) == sq_golden["specials/payload"].tobytes()
    # test_sq.py:107-111 frozen midpoints
    lut = oc.sq_lut(3, -4.0, 0.0)
    assert lut[6] == np.float32(2 ** -1.5) and lut[0] == np.float32(-(2 ** -0.5))
    # k = 1 midpoints (test_sq.py:114-117)
    l1 = oc.sq_lut(1, -4.0, 0.0)
    assert l1.tolist() == [np.float32(-0.25), np.float32(0.25)]


def test_bitpack_golden():
    # decode.test.ts:70-79: 0xE4 -> 2-bit [3, 2, 1, 0]
    assert oc.unpack_msb(bytes([0xE4]), 2, 4).tolist() == [3, 2, 1, 0]
    r = np.random.default_rng(0)
    for bits in range(1, 17):
        c = r.integers(0, 1 << bits, 37)
        assert oc.unpack_msb(oc.pack_msb(c, bits), bits, 37).tolist() == c.tolist()


# ------------------------------------------------------------------- VQ

def _books(z, name, d, width):
    ent = z[f"{name}/entries"]
    flat = z[f"{name}/books"]
    out, pos = [], 0
    for p, (lo, hi) in enumerate(oc.part_bounds(d, width)):
        cnt = int(ent[p]) * (hi - lo)
        out.append(flat[pos:pos + cnt].reshape(int(ent[p]), hi - lo))
        pos += cnt
    return out


VQ_CASES = ["cos_w4_L16", "euc_w4_L16", "cos_narrow", "euc_narrow", "cos_zeros",
            "cos_w4_L256", "euc_w8_L256", "lossless"]


@pytest.mark.parametrize("name", VQ_CASES)
def test_vq_oracle_assign_decode(vq_golden, name):
    z = vq_golden
    x = z[f"{name}/x"]
    w, L, metric_id = (int(v) for v in z[f"{name}/params"][:3])
    metric = ("euclidean", "cosine")[metric_id]
    books = _books(z, name, x.shape[1], w)
    assert np.array_equal(oc.vq_assign(x, books, w, metric), z[f"{name}/codes"])
    assert np.array_equal(oc.vq_assign(z[f"{name}/probe"], books, w, metric),
                          z[f"{name}/probe_codes"])
    assert np.array_equal(oc.vq_decode(z[f"{name}/codes"], books, x.shape[1], w),
                          z[f"{name}/decoded"])


@pytest.mark.parametrize("name", ["cos_w4_L16", "euc_w4_L16", "cos_narrow", "euc_narrow",
                                  "cos_zeros", "lossless"])
def test_vq_oracle_fit_is_bit_exact(vq_golden, name):
    z = vq_golden
    x = z[f"{name}/x"]
    w, L, metric_id, _layout, iters, restarts = (int(v) for v in z[f"{name}/params"])
    books, _ = oc.vq_fit(x, w, L, ("euclidean", "cosine")[metric_id], max_iters=iters,
                         restarts=restarts)
    ref = _books(z, name, x.shape[1], w)
    assert len(books) == len(ref)
    for a, b in zip(books, ref):
        assert np.array_equal(a, b)


# -------------------------------------------------------------- sampler

def _configs(z):
    out = []
    i = 0
    while f"cfg{i}/meta" in z.files:
        meta = z[f"cfg{i}/meta"]
        _, bs, seed, L = (int(v) for v in meta[:4])
        fans = tuple(int(v) for v in meta[4:4 + L])
        g = str(z[f"cfg{i}/graph"])
        out.append((i, g, fans, bs, seed))
        i += 1
    return out


def test_sampler_oracle_matches_reference(sampler_golden):
    z = sampler_golden
    for ci, gname, fans, bs, seed in _configs(z):
        off = z[f"graph/{gname}/row_offsets"]
        col = z[f"graph/{gname}/col_indices"]
        train = z[f"cfg{ci}/train"]
        batches, _ = sample_batches_oracle(off, col, train, fans, bs, seed)
        assert len(batches) == int(z[f"cfg{ci}/nbatches"])
        for bi, b in enumerate(batches):
            assert np.array_equal(b.seeds, z[f"cfg{ci}/b{bi}/seeds"])
            assert np.array_equal(b.frontier, z[f"cfg{ci}/b{bi}/frontier"])
            assert b.edges_touched == int(z[f"cfg{ci}/b{bi}/edges"])
            if bi < 3:
                for li, L in enumerate(b.layers):
                    assert np.array_equal(L.counts, z[f"cfg{ci}/b{bi}/l{li}/counts"])
                    assert np.array_equal(L.picks, z[f"cfg{ci}/b{bi}/l{li}/picks"])


def test_sampler_pcg_engine_equals_numpy_engine(sampler_golden):
    z = sampler_golden
    off = z["graph/pa2000/row_offsets"]
    col = z["graph/pa2000/col_indices"]
    a, sa = sample_batches_oracle(off, col, np.arange(300), (5, 3), 64, 11)
    b, sb = sample_batches_oracle(off, col, np.arange(300), (5, 3), 64, 11, engine="pcg")
    for x, y in zip(a, b):
        assert np.array_equal(x.frontier, y.frontier)
        for lx, ly in zip(x.layers, y.layers):
            assert np.array_equal(lx.picks, ly.picks)
    assert sa["state"]["state"] == sb["state"]["state"]


def test_row_source_oracle_equals_array_oracle(sampler_golden):
    """The row-source restatement (CSR rows served on demand, used for the
    full-size BASELINE graphs) gives the same batches, blocks and final
    stream state as the array oracle pinned to the reference above."""
    from oracle.sampler import HostRows, sample_batches_oracle_rows
    z = sampler_golden
    for ci, gname, fans, bs, seed in _configs(z):
        off = z[f"graph/{gname}/row_offsets"]
        col = z[f"graph/{gname}/col_indices"]
        train = z[f"cfg{ci}/train"]
        a, sa = sample_batches_oracle(off, col, train, fans, bs, seed)
        b, sb = sample_batches_oracle_rows(HostRows(off, col), off.size - 1, train, fans, bs,
                                           seed)
        assert len(a) == len(b)
        for x, y in zip(a, b):
            assert np.array_equal(x.seeds, y.seeds) and np.array_equal(x.frontier, y.frontier)
            assert x.edges_touched == y.edges_touched
            for lx, ly in zip(x.layers, y.layers):
                assert np.array_equal(lx.nodes, ly.nodes)
                assert np.array_equal(lx.counts, ly.counts)
                assert np.array_equal(lx.picks, ly.picks)
        assert sa == sb
