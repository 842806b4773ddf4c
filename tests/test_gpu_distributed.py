"""Row-partitioned evaluation end to end on the device: two ranks (two
processes sharing cuda:0, gloo for the combine) each run the GPU executor
on their shard (evaluate_sharded -> evaluate_partials -> combine_*); the
combined result must match the oracle on all rows."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
WORLD = 2
N = 100_003


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), LOCAL_RANK="0")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1709_06416_b200 import distributed as D
        from paper_1709_06416_b200 import workloads as W
        from weldmill.engine import Value
        comm = D.TorchComm()
        lo, hi = D.shard_bounds(N, rank, world)
        res = {}
        for name in ("q6", "blackscholes", "q1", "dict", "group", "hist"):
            wl = W.WORKLOADS[name]
            tree = W.compile_program(wl)
            types = W.input_types(wl)
            cols = W.host_columns(wl, hi - lo, row0=lo)
            env = {k: Value(types[k], v) for k, v in cols.items()}
            res[name] = D.evaluate_sharded(tree, env, None, W.externs_for(wl), comm, row0=lo)
        q.put((rank, res))
    except Exception as exc:  # surface the failure in the parent
        import traceback
        q.put((rank, traceback.format_exc()))
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
    out = dict(q.get(timeout=600) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        assert not isinstance(v, str), v
    return out


def _full(name):
    from paper_1709_06416_b200 import workloads as W
    from oracle import weld_oracle as O
    cols = W.host_columns(W.WORKLOADS[name], N)
    return O.ORACLES[name](cols)


def test_sharded_merger(results):
    want = _full("q6")
    for r in range(WORLD):
        got = results[r]["q6"][0]["values"][0]
        assert abs(got - want) <= 1e-9 * max(1.0, abs(want))


def test_sharded_appenders(results):
    call, put = _full("blackscholes")
    for r in range(WORLD):
        a, b = results[r]["blackscholes"]
        np.testing.assert_allclose(a["cols"][0], call, rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose(b["cols"][0], put, rtol=1e-9, atol=1e-9)


def test_sharded_q1_dict(results):
    want = _full("q1")
    got = results[0]["q1"][0]
    keys = list(zip(*[k.tolist() for k in got["keys"]]))
    assert keys == [k for k, _ in want]
    vals = list(zip(*[v.tolist() for v in got["vals"]]))
    for (_, wv), gv in zip(want, vals):
        assert gv[5] == wv[5]
        assert all(abs(a - b) <= 1e-9 * max(1.0, abs(a), abs(b)) for a, b in zip(gv[:5], wv[:5]))


def test_sharded_high_cardinality_dict(results):
    k, v = _full("dict")
    got = results[1]["dict"][0]
    np.testing.assert_array_equal(got["keys"][0], k)
    np.testing.assert_array_equal(got["vals"][0], v)


def test_sharded_group(results):
    ks, offs, vs = _full("group")
    want = {int(k): vs[offs[j]:offs[j + 1]].tolist() for j, k in enumerate(ks)}
    got = {}
    for r in range(WORLD):
        g = results[r]["group"][0]
        for j, k in enumerate(g["keys"][0]):
            got[int(k)] = g["vals"][0][g["offsets"][j]:g["offsets"][j + 1]].tolist()
    assert got == want


def test_sharded_vecmerger(results):
    want = _full("hist")
    for r in range(WORLD):
        np.testing.assert_allclose(results[r]["hist"][0]["cols"][0], want, rtol=1e-9, atol=1e-9)
