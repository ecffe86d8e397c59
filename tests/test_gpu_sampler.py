"""GPU sampler parity: bit-exact seeds, per-node picks (blocks), frontier,
edges_touched and final PCG64 stream state against the reference's golden
batches and the CPU oracle (which restates pipeline.py:185-222)."""

import numpy as np
import pytest
import torch

import paper_2207_14696_b200 as fg
from paper_2207_14696_b200.sampler import DeviceSampler
from oracle.sampler import sample_batches_oracle
from test_oracle import _configs

pytestmark = pytest.mark.gpu


def test_sample_batches_matches_reference_golden(sampler_golden):
    z = sampler_golden
    for ci, gname, fans, bs, seed in _configs(z):
        n = z[f"graph/{gname}/row_offsets"].size - 1
        g = fg.CsrGraph(n, z[f"graph/{gname}/row_offsets"], z[f"graph/{gname}/col_indices"])
        plan = fg.sample_batches(g, z[f"cfg{ci}/train"], fg.SamplerConfig(fans, bs, seed))
        assert plan.num_batches() == int(z[f"cfg{ci}/nbatches"])
        for bi, b in enumerate(plan.batches):
            assert np.array_equal(b.seeds, z[f"cfg{ci}/b{bi}/seeds"]), (ci, bi)
            assert np.array_equal(b.frontier, z[f"cfg{ci}/b{bi}/frontier"]), (ci, bi)
            assert b.edges_touched == int(z[f"cfg{ci}/b{bi}/edges"]), (ci, bi)


def _blocks(smp, sb, L):
    out = []
    for l in range(L):
        nn_ = int(sb.n_nodes[l].item())
        ip = sb.indptr[l][:nn_ + 1].cpu().numpy()
        np_ = int(sb.n_picks[l].item())
        out.append((sb.nodes[l][:nn_].cpu().numpy(), np.diff(ip),
                    sb.picks[l][:np_].cpu().numpy(),
                    None if sb.local[l] is None else sb.local[l][:np_].cpu().numpy()))
    return out


def test_device_sampler_blocks_match_golden(sampler_golden):
    z = sampler_golden
    for ci, gname, fans, bs, seed in _configs(z):
        n = z[f"graph/{gname}/row_offsets"].size - 1
        g = fg.CsrGraph(n, z[f"graph/{gname}/row_offsets"], z[f"graph/{gname}/col_indices"])
        smp = DeviceSampler(g.to_device(), fans, bs, need_local=True, unique_last=True)
        nb = smp.begin_epoch(z[f"cfg{ci}/train"], seed)
        for bi in range(min(3, nb)):
            sb = smp.sample(bi)
            for li, (nodes, counts, picks, local) in enumerate(_blocks(smp, sb, len(fans))):
                assert np.array_equal(counts, z[f"cfg{ci}/b{bi}/l{li}/counts"]), (ci, bi, li)
                assert np.array_equal(picks, z[f"cfg{ci}/b{bi}/l{li}/picks"]), (ci, bi, li)
                if local is not None:
                    nxt = sb.nodes[li + 1][:int(sb.n_nodes[li + 1].item())].cpu().numpy()
                    assert np.array_equal(nxt[local], picks)
        smp.check_errors()


def _powerlaw_graph(n, seed):
    from paper_2207_14696_b200.synth import generate_graph
    dg, labels = generate_graph(n, 30.0, 8, seed=seed)
    return dg


def test_device_sampler_matches_oracle_on_products_like_graph():
    dg = _powerlaw_graph(120_000, 3)
    host = dg.to_host()
    train = np.arange(0, 120_000, 37)
    fans, bs, seed = (15, 10, 5), 1024, 4
    smp = DeviceSampler(dg, fans, bs, need_local=True, want_frontier=True)
    smp.begin_epoch(train, seed)
    ref, ref_state = sample_batches_oracle(host.row_offsets, host.col_indices, train, fans, bs,
                                           seed, max_batches=2)
    for bi, rb in enumerate(ref):
        sb = smp.sample(bi)
        got = _blocks(smp, sb, len(fans))
        for li, L in enumerate(rb.layers):
            assert np.array_equal(got[li][0], L.nodes)
            assert np.array_equal(got[li][1], L.counts)
            assert np.array_equal(got[li][2], L.picks)
        nf = int(sb.n_frontier.item())
        assert np.array_equal(sb.frontier[:nf].cpu().numpy(), rb.frontier)
    st = smp.stream_state()
    assert st["state"]["state"] == ref_state["state"]["state"]
    assert st["has_uint32"] == ref_state["has_uint32"]
    smp.check_errors()


def _seeds_with_hub_rejection(n_train, hubs, deg, fanout, want=2, limit=3000):
    """Seeds whose stream rejects at least one Lemire draw while sampling
    the hubs (which come first in the sorted layer), found with the oracle
    PCG64 restatement."""
    from oracle.pcg64 import Pcg64Stream
    found = []
    for seed in range(limit):
        rng = np.random.default_rng(seed)
        rng.permutation(np.arange(n_train))
        st = Pcg64Stream.from_numpy(rng.bit_generator.state)
        for _ in range(hubs):
            st.choice_noreplace(deg, fanout)
        if st.draws32 > hubs * (2 * fanout - 1):
            found.append(seed)
            if len(found) == want:
                break
    return found


@pytest.mark.parametrize("fanout,seeds,n_leaves", [(200, 40, 0), (16, 60, 0), (8, 120, 0),
                                                    (5, None, 33000)])
def test_sampler_lemire_rejection_fixup(fanout, seeds, n_leaves):
    """Hubs of degree ~3e6 make Lemire rejections likely (p ~ 5e-4 per
    draw); every rejection shifts all later stream offsets of the layer, which
    the fix-up must repair for the picks to stay bit-exact.  fanout 200 runs
    the thread-per-node path, 16 and 8 the lane-group paths (G = 32 / 16);
    with 40k extra leaf seeds the layer is large enough for the register
    thread path (F = 5)."""
    hubs, deg = 6, 3_000_017
    n = hubs + deg
    # bipartite: hub h connects to all leaves; leaves connect to all hubs
    off = [0]
    cols = []
    leaves = np.arange(hubs, n, dtype=np.int32)
    for h in range(hubs):
        c = np.concatenate([[h], leaves]).astype(np.int32)
        cols.append(c)
        off.append(off[-1] + c.size)
    leaf_nb = np.arange(hubs, dtype=np.int32)
    leaf_cols = np.empty((deg, hubs + 1), np.int32)
    leaf_cols[:, :hubs] = leaf_nb[None, :]
    leaf_cols[:, hubs] = leaves
    cols.append(leaf_cols.reshape(-1))
    off = np.concatenate([np.array(off, np.int64),
                          off[-1] + (hubs + 1) * np.arange(1, deg + 1, dtype=np.int64)])
    col = np.concatenate(cols)
    g = fg.CsrGraph.trusted(n, off, col, True)
    dg = g.to_device()
    train = np.arange(hubs + n_leaves)
    bs = train.size
    fans = (fanout,)
    total_rej = 0
    seed_list = range(seeds) if seeds else _seeds_with_hub_rejection(bs, hubs, deg + 1, fanout)
    for seed in seed_list:
        smp = DeviceSampler(dg, fans, bs, need_local=False, want_frontier=True)
        smp.begin_epoch(train, seed)
        ref, ref_state = sample_batches_oracle(off, col, train, fans, bs, seed)
        sb = smp.sample(0)
        np_ = int(sb.n_picks[0].item())
        assert np.array_equal(sb.picks[0][:np_].cpu().numpy(), ref[0].layers[0].picks), seed
        st = smp.stream_state()
        assert st["state"]["state"] == ref_state["state"]["state"], seed
        draws = int(smp.rng[6].item())
        total_rej += draws - (hubs + n_leaves) * (2 * fanout - 1)
    assert total_rej > 0, "no Lemire rejection exercised"


@pytest.mark.parametrize("fans,bs", [((1,), 7), ((3, 2), 64), ((4, 4, 4), 1000)])
def test_sampler_edge_cases_match_oracle(fans, bs):
    """No self-loops with isolated (degree-0) nodes, duplicate train ids
    (np.unique), a partial last batch, fanout 1, a batch larger than the
    train set: per-node picks, frontier and final stream state equal the
    oracle restatement of pipeline.py:185-222."""
    r = np.random.default_rng(len(fans) * 100 + bs)
    n = 3000
    src = r.integers(0, n - 200, 12_000)          # nodes n-200.. are isolated
    dst = r.integers(0, n - 200, 12_000)
    keep = src != dst
    a = np.concatenate([src[keep], dst[keep]])
    b = np.concatenate([dst[keep], src[keep]])
    key = np.unique(a.astype(np.int64) * n + b)
    rows, cols = key // n, (key % n).astype(np.int32)
    off = np.zeros(n + 1, np.int64)
    np.add.at(off, rows + 1, 1)
    off = np.cumsum(off)
    g = fg.CsrGraph(n, off, cols)
    train = np.concatenate([r.integers(0, n, 400), np.arange(n - 50, n)])  # dups + isolated
    seed = 11
    smp = DeviceSampler(g.to_device(), fans, bs, need_local=True, want_frontier=True)
    nb = smp.begin_epoch(train, seed)
    ref, ref_state = sample_batches_oracle(off, cols, train, fans, bs, seed)
    assert nb == len(ref)
    for bi, rb in enumerate(ref):
        sb = smp.sample(bi)
        got = _blocks(smp, sb, len(fans))
        for li, L in enumerate(rb.layers):
            assert np.array_equal(got[li][0], L.nodes), (bi, li)
            assert np.array_equal(got[li][1], L.counts), (bi, li)
            assert np.array_equal(got[li][2], L.picks), (bi, li)
        nf = int(sb.n_frontier.item())
        assert np.array_equal(sb.frontier[:nf].cpu().numpy(), rb.frontier)
    st = smp.stream_state()
    assert st["state"]["state"] == ref_state["state"]["state"]
    smp.check_errors()


def test_sampler_fanout_above_200_small_graph():
    """Fanouts above 200 are accepted (no blanket cap): on degrees <= 10000
    numpy's choice stays on the Floyd branch, so picks and the stream state
    equal the oracle.  A hub with deg > 10000 and f > deg // 50 would take
    numpy's partial Fisher-Yates branch: that is reported as a DataError."""
    n = 1500
    r = np.random.default_rng(5)
    key = set()
    for u in range(n):
        for v in r.choice(n, 400, replace=False):
            if u != v:
                key.add((u, int(v)))
                key.add((int(v), u))
    key |= {(u, u) for u in range(n)}
    key = np.array(sorted(key), np.int64)
    off = np.zeros(n + 1, np.int64)
    np.add.at(off, key[:, 0] + 1, 1)
    off = np.cumsum(off)
    col = key[:, 1].astype(np.int32)
    g = fg.CsrGraph(n, off, col)
    train = np.arange(0, n, 3)
    fans, bs, seed = (300, 2), 128, 9
    smp = DeviceSampler(g.to_device(), fans, bs, need_local=True, want_frontier=True)
    smp.begin_epoch(train, seed)
    ref, ref_state = sample_batches_oracle(off, col, train, fans, bs, seed, max_batches=2)
    for bi, rb in enumerate(ref):
        sb = smp.sample(bi)
        got = _blocks(smp, sb, len(fans))
        for li, L in enumerate(rb.layers):
            assert np.array_equal(got[li][2], L.picks), (bi, li)
    assert smp.stream_state()["state"]["state"] == ref_state["state"]["state"]
    smp.check_errors()
    # hub of degree 12000 with fanout 300 > 12000 // 50: numpy's other branch
    hub_deg = 12_000
    n2 = hub_deg + 1
    off2 = np.concatenate([[0, hub_deg + 1], hub_deg + 1 + 2 * np.arange(1, hub_deg + 1)])
    col2 = np.concatenate([np.arange(n2), np.stack([np.zeros(hub_deg), np.arange(1, n2)],
                                                   1).reshape(-1)]).astype(np.int32)
    g2 = fg.CsrGraph(n2, off2.astype(np.int64), col2)
    smp2 = DeviceSampler(g2.to_device(), (300,), 4, need_local=False)
    smp2.begin_epoch(np.array([0]), 1)
    smp2.sample(0)
    with pytest.raises(fg.DataError):
        smp2.check_errors()


@pytest.mark.parametrize("cap,live,n", [(1024, 1024, 111_059_956), (1024, 700, 50_000_000),
                                        (4096, 4096, 244_160_499), (3000, 1, 2 ** 30),
                                        (1, 1, 5)])
def test_seed_sort_equals_numpy_sort(cap, live, n):
    """fg_sort_ids (the seed layer on graphs past 2^24 nodes) is np.sort of
    the batch's ids (pipeline.py:203), duplicates kept; count from the
    device scalar."""
    from paper_2207_14696_b200 import _native as N
    rng = np.random.default_rng(cap + live)
    ids = rng.integers(0, n, cap).astype(np.int64)
    ids[: live // 3] = ids[0]  # duplicates
    d_ids = torch.from_numpy(ids).cuda()
    out = torch.full((cap,), -7, dtype=torch.int32, device="cuda")
    cnt = torch.tensor([live], dtype=torch.int64, device="cuda")
    ocnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    N.call("fg_sort_ids", N.ptr(d_ids), N.ptr(cnt), cap, N.ptr(out), N.ptr(ocnt), n,
           N.stream_handle())
    assert int(ocnt.item()) == live
    o = out.cpu().numpy()
    assert np.array_equal(o[:live], np.sort(ids[:live]).astype(np.int32))
    assert (o[live:] == -7).all()
