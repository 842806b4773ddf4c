"""Multi-rank combine logic (paper_1709_06416_b200/distributed.py) over
torch.distributed gloo, world_size 2, on CPU.  Per-rank partials come from
the numpy oracle on each rank's row shard; the combined result must equal
the oracle on all rows (bit-exact for integers, 1e-9 for f64)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1709_06416_b200 import distributed as D
        from paper_1709_06416_b200 import workloads as W
        from oracle import weld_oracle as O
        comm = D.TorchComm()
        res = {}
        n = 5003
        lo, hi = D.shard_bounds(n, rank, world)
        # merger: Q6 partial sums per rank, folded in rank order
        q6 = W.host_columns(W.WORKLOADS["q6"], hi - lo, row0=lo)
        part = O.q6(q6)
        vals, has = D.combine_merger([part], hi > lo, "+", ["f64"], comm)
        res["q6"] = vals[0]
        # merger min with NaN rules, i64 wrap
        vals, _ = D.combine_merger([float("nan") if rank == 0 else 2.5], True, "min", ["f64"], comm)
        res["fmin"] = vals[0]
        vals, _ = D.combine_merger([2**62 + rank], True, "+", ["i64"], comm)
        res["wrap"] = vals[0]
        vals, has = D.combine_merger([0.0], False, "+", ["f64"], comm)
        res["empty"] = (vals[0], has)
        # appender: ordered gather of Black-Scholes outputs
        bs = W.host_columns(W.WORKLOADS["blackscholes"], hi - lo, row0=lo)
        call, put = O.blackscholes(bs)
        res["bs"] = D.combine_appender([call, put], comm)
        # dictmerger: hash-partitioned all-to-all + keyed fold + gather
        dc = W.host_columns(W.WORKLOADS["dict"], hi - lo, row0=lo)
        dc["k"] = dc["k"] % 97            # force cross-rank key collisions
        k, v = O.dict_sum(dc)
        pk, pv = D.combine_dict([k], [v], "+", ["i64"], comm)
        gk, gv = D.gather_partitions(pk, pv, comm)
        res["dict"] = (gk[0], gv[0])
        # groupbuilder: per-key input order across ranks
        gk_, offs, gvals = D.combine_group([dc["k"]], [dc["v"]], comm)
        res["group"] = (comm.allgather(gk_[0]), comm.allgather(offs), comm.allgather(gvals[0]))
        # vecmerger: init counted once
        hc = W.host_columns(W.WORKLOADS["hist"], hi - lo, row0=lo)
        bins = np.arange(1000, dtype=np.float64)
        start = D.vecmerger_start([bins], "+", ["f64"], rank)[0]
        local = start + np.bincount(hc["idx"] % 1000, weights=hc["w"], minlength=1000)
        res["hist"] = D.combine_vecmerger([local], "+", ["f64"], comm)[0]
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
    return out


def test_merger_combine(results):
    from paper_1709_06416_b200 import workloads as W
    from oracle import weld_oracle as O
    want = O.q6(W.host_columns(W.WORKLOADS["q6"], 5003))
    for r in range(WORLD):
        got = results[r]["q6"]
        assert abs(got - want) <= 1e-9 * max(1.0, abs(want))
        assert results[r]["fmin"] == 2.5                      # min prefers numbers over NaN
        assert results[r]["wrap"] == (2**62 * 2 + 1) - 2**64  # i64 wraps
        assert results[r]["empty"] == (0.0, False)            # identity when no rank merged


def test_appender_ordered_gather(results):
    from paper_1709_06416_b200 import workloads as W
    from oracle import weld_oracle as O
    call, put = O.blackscholes(W.host_columns(W.WORKLOADS["blackscholes"], 5003))
    for r in range(WORLD):
        gc, gp = results[r]["bs"]
        np.testing.assert_array_equal(gc, call)
        np.testing.assert_array_equal(gp, put)


def test_dict_all_to_all(results):
    from paper_1709_06416_b200 import workloads as W
    from oracle import weld_oracle as O
    dc = W.host_columns(W.WORKLOADS["dict"], 5003)
    dc["k"] = dc["k"] % 97
    k, v = O.dict_sum(dc)
    for r in range(WORLD):
        gk, gv = results[r]["dict"]
        np.testing.assert_array_equal(gk, k)
        np.testing.assert_array_equal(gv, v)


def test_group_preserves_order_across_ranks(results):
    from paper_1709_06416_b200 import workloads as W
    from oracle import weld_oracle as O
    dc = W.host_columns(W.WORKLOADS["dict"], 5003)
    dc["k"] = dc["k"] % 97
    ks, offs, vs = O.group(dc)
    want = {int(k): vs[offs[j]:offs[j + 1]].tolist() for j, k in enumerate(ks)}
    got = {}
    keys, offsets, vals = results[0]["group"]
    for kk, oo, vv in zip(keys, offsets, vals):
        for j, k in enumerate(kk):
            got[int(k)] = vv[oo[j]:oo[j + 1]].tolist()
    assert got == want


def test_vecmerger_init_counted_once(results):
    from paper_1709_06416_b200 import workloads as W
    hc = W.host_columns(W.WORKLOADS["hist"], 5003)
    want = np.arange(1000, dtype=np.float64) + np.bincount(hc["idx"] % 1000, weights=hc["w"], minlength=1000)
    for r in range(WORLD):
        np.testing.assert_allclose(results[r]["hist"], want, rtol=1e-12)


def test_shard_bounds_cover_rows():
    from paper_1709_06416_b200 import distributed as D
    for n in (0, 1, 7, 5003):
        for w in (1, 2, 3, 8):
            spans = [D.shard_bounds(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
