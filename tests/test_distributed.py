"""The multi-rank combine protocol of paper_1709_06416_b200/distributed.py
over torch.distributed gloo on CPU (world_size 2 and 3).

What runs here is the host side of the protocol exactly as the device path
uses it -- shard bounds, order keys, sampled splitters, the exchange plan,
vecmerger slices, and StagedComm's host collectives -- with numpy standing
in for the three device kernels (wg_partition's stable range split, the
rank-order fold kernels, and the local dictmerger / groupbuilder).  The
combined results must equal the oracle on all rows: bit-exact for integers
and order, 1e-9 for f64.  The device kernels themselves are covered by
tests/test_gpu_distributed.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# --- numpy stand-ins for the device kernels --------------------------------


def _partition(keys, others, split):
    """wg_partition: dest = #splitters <= okey(first key leaf); stable."""
    from paper_1709_06416_b200 import distributed as D
    ok = D.okey_np(keys[0], "i64" if keys[0].dtype.kind == "i" else "f64")
    dest = np.searchsorted(split, ok, side="right")
    order = np.argsort(dest, kind="stable")
    counts = np.bincount(dest, minlength=len(split) + 1)
    return [c[order] for c in keys], [c[order] for c in others], counts


def _alltoallv(comm, col, send, soff, recv, roff):
    parts = [col[soff[d]:soff[d] + send[d]] for d in range(comm.world)]
    # every rank's part for me, via the host all-gather (gloo)
    got = comm.allgather_host(np.concatenate(parts) if parts else col[:0])
    sends = comm.allgather_host(np.asarray(send, dtype=np.int64))
    out = []
    for s in range(comm.world):
        off = int(np.sum(sends[s][:comm.rank]))
        out.append(got[s][off:off + int(sends[s][comm.rank])])
    res = np.concatenate(out)
    assert res.size == int(np.sum(recv))
    return res


def _exchange(comm, keys, others):
    from paper_1709_06416_b200 import distributed as D
    n = keys[0].size
    samp = D.okey_np(keys[0][D.sample_positions(n)], "i64")
    split = D.choose_splitters(comm.allgather_host(samp), comm.world)
    pk, po, counts = _partition(keys, others, split)
    mat = np.stack(comm.allgather_host(counts.astype(np.int64)))
    send, soff, recv, roff = D.exchange_plan(mat, comm.rank)
    return ([_alltoallv(comm, c, send, soff, recv, roff) for c in pk],
            [_alltoallv(comm, c, send, soff, recv, roff) for c in po])


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1709_06416_b200 import distributed as D
        from paper_1709_06416_b200 import workloads as W
        from paper_1709_06416_b200.semantics import fold
        from oracle import weld_oracle as O
        comm = D.StagedComm()
        res = {}
        n = 5003
        lo, hi = D.shard_bounds(n, rank, world)
        # merger: slots (value, merged flag) all-gathered, folded in rank order
        q6 = W.host_columns(W.WORKLOADS["q6"], hi - lo, row0=lo)

        def merger(val, has, op, kind):
            slots = comm.allgather_host(np.array([val, 1.0 if has else 0.0]))
            acc, seen = None, False
            for s in slots:
                if s[1]:
                    acc = s[0] if not seen else fold(op, kind, acc, s[0])
                    seen = True
            return acc, seen

        res["q6"] = merger(O.q6(q6), hi > lo, "+", "f64")[0]
        res["fmin"] = merger(float("nan") if rank == 0 else 2.5, True, "min", "f64")[0]
        res["empty"] = merger(0.0, False, "+", "f64")[1]
        # appender: counts all-gathered -> offsets; the rank-order concatenation is the result
        bs = W.host_columns(W.WORKLOADS["blackscholes"], hi - lo, row0=lo)
        call, put = O.blackscholes(bs)
        counts = np.concatenate(comm.allgather_host(np.array([call.size], dtype=np.int64)))
        res["bs_offset"] = (int(counts[:rank].sum()), int(counts.sum()))
        res["bs"] = [np.concatenate(comm.allgather_host(c)) for c in (call, put)]
        # dictmerger: local aggregate -> range partition -> exchange -> local merge
        dc = W.host_columns(W.WORKLOADS["dict"], hi - lo, row0=lo)
        dc["k"] = dc["k"] % 97 - 40          # cross-rank collisions, negative keys
        k, v = O.dict_sum(dc)
        (rk,), (rv,) = _exchange(comm, [k], [v])
        mk, mv = O.dict_sum({"k": rk, "v": rv})
        res["dict"] = (np.concatenate(comm.allgather_host(mk)), np.concatenate(comm.allgather_host(mv)))
        # groupbuilder: rows in local order -> exchange -> groups in source-rank order
        (gk,), (gv,) = _exchange(comm, [dc["k"]], [dc["v"]])
        ks, offs, vs = O.group({"k": gk, "v": gv})
        res["group"] = (comm.allgather_host(ks), comm.allgather_host(offs), comm.allgather_host(vs))
        # vecmerger: slices all-to-all, rank-order fold, all-gather of the folded slices
        hc = W.host_columns(W.WORKLOADS["hist"], hi - lo, row0=lo)
        nb = 1001
        bins = np.arange(nb, dtype=np.float64) if rank == 0 else np.zeros(nb)
        local = bins + np.bincount(hc["idx"] % nb, weights=hc["w"], minlength=nb)
        sl = D.slice_bounds(nb, world)
        send = np.array([b - a for a, b in sl], dtype=np.int64)
        soff = np.array([a for a, _ in sl], dtype=np.int64)
        L = int(send[rank])
        chunks = _alltoallv(comm, local, send, soff, np.full(world, L), np.arange(world) * L)
        mine = chunks[:L].copy()
        for s in range(1, world):
            mine = mine + chunks[s * L:(s + 1) * L]
        res["hist"] = np.concatenate(comm.allgather_host(mine))
        q.put((rank, res))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module", params=[2, 3])
def run(request):
    world = request.param
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        assert not isinstance(v, str), v
    return world, out


def test_merger_combine(run):
    from paper_1709_06416_b200 import workloads as W
    from oracle import weld_oracle as O
    world, results = run
    want = O.q6(W.host_columns(W.WORKLOADS["q6"], 5003))
    for r in range(world):
        got = results[r]["q6"]
        assert abs(got - want) <= 1e-9 * max(1.0, abs(want))
        assert results[r]["fmin"] == 2.5                      # min prefers numbers over NaN
        assert results[r]["empty"] is False                   # identity when no rank merged


def test_appender_ordered_gather(run):
    from paper_1709_06416_b200 import workloads as W
    from oracle import weld_oracle as O
    world, results = run
    call, put = O.blackscholes(W.host_columns(W.WORKLOADS["blackscholes"], 5003))
    for r in range(world):
        gc, gp = results[r]["bs"]
        np.testing.assert_array_equal(gc, call)
        np.testing.assert_array_equal(gp, put)
    offs = [results[r]["bs_offset"] for r in range(world)]
    assert offs[0][0] == 0 and all(o[1] == 5003 for o in offs)


def test_dict_range_partition_is_globally_sorted(run):
    from paper_1709_06416_b200 import workloads as W
    from oracle import weld_oracle as O
    world, results = run
    dc = W.host_columns(W.WORKLOADS["dict"], 5003)
    dc["k"] = dc["k"] % 97 - 40
    k, v = O.dict_sum(dc)
    for r in range(world):
        gk, gv = results[r]["dict"]
        np.testing.assert_array_equal(gk, k)           # rank-order concatenation is sorted
        np.testing.assert_array_equal(gv, v)


def test_group_preserves_order_across_ranks(run):
    from paper_1709_06416_b200 import workloads as W
    from oracle import weld_oracle as O
    world, results = run
    dc = W.host_columns(W.WORKLOADS["dict"], 5003)
    dc["k"] = dc["k"] % 97 - 40
    ks, offs, vs = O.group(dc)
    keys, offsets, vals = results[0]["group"]
    gk = np.concatenate(keys)
    np.testing.assert_array_equal(gk, ks)
    got = {}
    for kk, oo, vv in zip(keys, offsets, vals):
        for j, key in enumerate(kk):
            got[int(key)] = vv[oo[j]:oo[j + 1]].tolist()
    assert got == {int(key): vs[offs[j]:offs[j + 1]].tolist() for j, key in enumerate(ks)}


def test_vecmerger_init_counted_once(run):
    from paper_1709_06416_b200 import workloads as W
    world, results = run
    hc = W.host_columns(W.WORKLOADS["hist"], 5003)
    nb = 1001
    want = np.arange(nb, dtype=np.float64) + np.bincount(hc["idx"] % nb, weights=hc["w"], minlength=nb)
    for r in range(world):
        np.testing.assert_allclose(results[r]["hist"], want, rtol=1e-12)


def test_shard_bounds_cover_rows():
    from paper_1709_06416_b200 import distributed as D
    for n in (0, 1, 7, 5003):
        for w in (1, 2, 3, 8):
            spans = [D.shard_bounds(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_okey_np_matches_order_key():
    """The splitters' order keys sort like the reference's order_key
    (builders.py:496-507): signed ints, floats with -0.0 == 0.0, NaN last."""
    from paper_1709_06416_b200 import distributed as D
    from weldmill.engine.builders import order_key
    ints = np.array([5, -3, 0, -(1 << 63), (1 << 63) - 1, 7], dtype=np.int64)
    assert np.argsort(D.okey_np(ints, "i64"), kind="stable").tolist() == \
        sorted(range(len(ints)), key=lambda j: order_key(int(ints[j])))
    fl = np.array([1.5, -0.0, 0.0, float("nan"), -float("inf"), float("inf"), -2.0])
    ok = D.okey_np(fl, "f64")
    assert ok[1] == ok[2]                                 # -0.0 and 0.0 are one key
    assert ok[3] == ok.max() and ok[3] > ok[5]            # NaN after +inf
    assert np.argsort(ok[[0, 4, 5, 6]]).tolist() == [1, 3, 0, 2]


def test_splitters_balance_and_cover():
    from paper_1709_06416_b200 import distributed as D
    rng = np.random.default_rng(1)
    samples = [np.sort(rng.integers(0, 1 << 60, 256).astype(np.uint64)) for _ in range(4)]
    sp = D.choose_splitters(samples, 4)
    assert sp.size == 3 and np.all(np.diff(sp.astype(np.float64)) >= 0)
    allk = np.concatenate(samples)
    share = np.bincount(np.searchsorted(sp, allk, side="right"), minlength=4) / allk.size
    assert share.min() > 0.2
    assert D.choose_splitters(samples, 1).size == 0


def test_exchange_plan_layout():
    from paper_1709_06416_b200 import distributed as D
    mat = np.array([[3, 1, 0], [2, 2, 2], [0, 0, 5]])
    send, soff, recv, roff = D.exchange_plan(mat, 1)
    assert send.tolist() == [2, 2, 2] and soff.tolist() == [0, 2, 4]
    assert recv.tolist() == [1, 2, 0] and roff.tolist() == [0, 1, 3]
