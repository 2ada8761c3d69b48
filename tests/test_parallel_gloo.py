"""The multi-GPU host logic on CPU: world_size-2 gloo process groups, oracle-made inputs.

Checks that sharding covers every global path once and that combining two ranks' norms
gives the single-process reference numbers (Err bitwise, ME/moments to rounding)."""
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


def test_shard_covers_all_paths():
    from paper_2207_09776_b200.parallel import shard
    for M in (1, 7, 16, 16384, 131072):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                off, cnt = shard(M, r, world)
                seen += list(range(off, off + cnt))
            assert seen == list(range(M))


def _problem():
    """Per-path relative errors / ME / moments of a small exact-vs-perturbed ensemble."""
    from oracle import restate as rs
    d, M, T, dt_leb = 12, 7, 0.2, 1e-3
    values, _ = rs.simulate_brownian(T, dt_leb, M, 5)
    h = 8.0 / (d + 1)
    nodes = np.array([-4.0 + (i + 1) * h for i in range(d)])
    ref = np.stack([rs.exact_field(nodes, nodes, T, 1.1, 1 / np.sqrt(10), *rs.functionals(values[m], 0, 200, dt_leb)[1:3])
                    for m in range(M)])
    rng = np.random.default_rng(3)
    app = ref * (1 + 1e-3 * rng.standard_normal(ref.shape))
    status = np.zeros(M, np.uint8)
    return d, M, ref, app, status


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2207_09776_b200.parallel import combine_error_stats, max_over_ranks, shard
    from oracle import restate as rs
    d, M, ref, app, status = _problem()
    off, cnt = shard(M, rank, world)
    lo, hi = rs.central_region(d, 1)
    rel = []
    for m in range(off, off + cnt):
        r, a = ref[m].reshape(d, d), app[m].reshape(d, d)  # [j][i]
        num = den = 0.0
        for j in range(lo, hi + 1):
            for i in range(lo, hi + 1):
                num += (r[j, i] - a[j, i]) ** 2
                den += r[j, i] ** 2
        rel.append(np.sqrt(num) / np.sqrt(den))
    local = rs.errors(d, 1, ref[off:off + cnt], app[off:off + cnt])
    mom = np.concatenate([app[off:off + cnt].sum(0), (app[off:off + cnt] ** 2).sum(0)])
    out = combine_error_stats(np.array(rel), local["me"], cnt - local["excluded"], local["blowups"], M,
                              moments=mom)
    mx = max_over_ranks(float(rank + 1))
    if rank == 0:
        q.put((out["err"], out["me"], out["sum_u"], mx))
    dist.destroy_process_group()


def test_combine_two_ranks_matches_single_process():
    from oracle import restate as rs
    d, M, ref, app, status = _problem()
    want = rs.errors(d, 1, ref, app)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err, me, sum_u, mx = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err == want["err"]  # bitwise: per-path ratios summed in global path order
    assert np.allclose(me, want["me"], rtol=1e-14, atol=0)
    assert np.allclose(sum_u, app.sum(0), rtol=1e-14)
    assert mx == 2.0


def test_blowups_force_infinite_err():
    from paper_2207_09776_b200.parallel import combine_error_stats
    out = combine_error_stats(np.array([0.1, np.nan, 0.2]), np.ones((2, 2)), 2, 1, 3)
    assert out["err"] == np.inf and out["blowups"] == 1


def test_c_abi_shard_equals_python_shard(s2b):
    from paper_2207_09776_b200.parallel import shard
    for M in (1, 7, 16384, 131072):
        for world in (1, 2, 3, 8):
            for r in range(world):
                assert s2b.shard(M, r, world) == shard(M, r, world)


def _e2e_problem():
    d, M, T, dt_leb, order, dt_steps = 10, 5, 0.2, 1e-3, 2, 100
    return d, M, T, dt_leb, order, dt_steps


def _e2e_worker(rank, world, port, q):
    """One rank end to end on CPU: its shard of the global paths (streams keyed by the global
    path id, so a slice of the global batch), the oracle's Magnus solve of each of its paths,
    its norms against the closed form, and the one combine of the statistics."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2207_09776_b200 as s2b
    from paper_2207_09776_b200.parallel import combine_error_stats, shard
    from oracle import restate as rs
    d, M, T, dt_leb, order, dt_steps = _e2e_problem()
    off, cnt = shard(M, rank, world)
    values = s2b.simulate_brownian(T, dt_leb, M, 77)[off:off + cnt]  # = trajectories off..off+cnt-1
    host = s2b.HostOps(s2b.GridSpec.square(d), "langevin-constant", order=order)
    phi = s2b.gaussian_datum(s2b.GridSpec.square(d))
    total = int(round(T / dt_leb))
    h = 8.0 / (d + 1)
    nodes = np.array([-4.0 + (i + 1) * h for i in range(d)])
    app, ref = [], []
    for m in range(cnt):
        st, status, _, _ = rs.magnus_path(d * d, order, host.sources(), phi, values[m], dt_leb, dt_steps, total, [total])
        app.append(st[0])
        W, IW = rs.functionals(values[m], 0, total, dt_leb)[1:3]
        ref.append(rs.exact_field(nodes, nodes, T, 1.1, 1 / np.sqrt(10), W, IW))
    app, ref = np.array(app), np.array(ref)
    local = rs.errors(d, 1, ref, app)
    lo, hi = rs.central_region(d, 1)
    rel = []
    for m in range(cnt):
        r, a = ref[m].reshape(d, d), app[m].reshape(d, d)
        num = den = 0.0
        for j in range(lo, hi + 1):
            for i in range(lo, hi + 1):
                num += (r[j, i] - a[j, i]) ** 2
                den += r[j, i] ** 2
        rel.append(np.sqrt(num) / np.sqrt(den))
    mom = np.concatenate([app.sum(0), (app ** 2).sum(0)])
    out = combine_error_stats(np.array(rel), local["me"], cnt - local["excluded"], local["blowups"], M, moments=mom)
    if rank == 0:
        q.put((out["err"], out["me"], out["sum_u"], app))
    else:
        q.put((None, None, None, app))
    dist.destroy_process_group()


def test_two_ranks_end_to_end_match_one_process():
    """Sharding + per-path streams + combine, end to end on two gloo ranks: Err bitwise, ME and
    moments to rounding, and every rank's solutions are the single-process ones."""
    import paper_2207_09776_b200 as s2b
    from oracle import restate as rs
    d, M, T, dt_leb, order, dt_steps = _e2e_problem()
    values = s2b.simulate_brownian(T, dt_leb, M, 77)
    host = s2b.HostOps(s2b.GridSpec.square(d), "langevin-constant", order=order)
    phi = s2b.gaussian_datum(s2b.GridSpec.square(d))
    total = int(round(T / dt_leb))
    h = 8.0 / (d + 1)
    nodes = np.array([-4.0 + (i + 1) * h for i in range(d)])
    app = np.array([rs.magnus_path(d * d, order, host.sources(), phi, values[m], dt_leb, dt_steps, total, [total])[0][0]
                    for m in range(M)])
    ref = np.array([rs.exact_field(nodes, nodes, T, 1.1, 1 / np.sqrt(10), *rs.functionals(values[m], 0, total, dt_leb)[1:3])
                    for m in range(M)])
    want = rs.errors(d, 1, ref, app)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_e2e_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    err, me, sum_u, _ = next(g for g in got if g[0] is not None)
    apps = sorted((g[3] for g in got), key=len, reverse=True)  # rank 0 holds the first (larger) range
    assert np.array_equal(np.concatenate(apps), app)
    assert err == want["err"]
    assert np.allclose(me, want["me"], rtol=1e-14, atol=0)
    assert np.allclose(sum_u, app.sum(0), rtol=1e-14)
