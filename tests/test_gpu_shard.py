"""Row-sharded operators on the GPU: two ranks share cuda:0 over gloo.

NCCL refuses two ranks on one device, and the test box has one GPU, so the
collectives run on gloo (staged through host memory) while every kernel --
halo packing, the ghost-aware tiled SpMM, the diagonal constraint pass, the
fused ALM update -- runs on the device exactly as under NCCL.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, deg, ld, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2407_15049_b200 import alm, linops, problem, shard
        from paper_2407_15049_b200.device import Device
        dev = Device()
        dev.world = world
        ops = shard.sharded_maxcut_ops(n, deg, 11, rank, world, dev)
        rng = np.random.default_rng(5)
        Rg = rng.standard_normal((n, ld))
        Rl = torch.as_tensor(Rg[ops.lo:ops.hi]).cuda().contiguous()
        core = alm.AlmCore(ops, ops.hi - ops.lo, ld)
        core.constraint_values(Rl)
        core.c_times(Rl, core.CR)
        lam = torch.zeros(ops.hi - ops.lo, dtype=torch.float64, device="cuda")
        g = torch.empty_like(Rl)
        y = torch.empty_like(Rl)
        zero = torch.zeros_like(Rl)
        out = core.grad_value(Rl, lam, 3.0, 1.0, zero, g, y, [], refresh=True)
        # global reference on rank 0's view: same edges, single-process operators
        eu, ev = shard.random_graph_edges(n, deg, 11, torch.device("cuda"))
        p = problem.build_maxcut(problem.GraphEdgeList(n, eu.cpu().numpy(), ev.cpu().numpy(),
                                                      np.ones(eu.numel())))
        ref = linops.build_operators(p, dev=Device())
        CR = linops.spmm(ref.c_mat, Rg)
        err = float(np.abs(core.CR.cpu().numpy() - CR[ops.lo:ops.hi]).max() / (1 + np.abs(CR).max()))
        ax = np.einsum("ij,ij->i", Rg, Rg)
        axe = float(np.abs(core.ax.cpu().numpy() - ax[ops.lo:ops.hi]).max())
        w = 3.0 * (ax - 1.0)
        G = 2.0 * (w[:, None] * Rg + CR)
        q.put((rank, err, axe, float(out["gg"]), float(np.sum(G * G)), float(out["crr"]),
               float(np.sum(CR * Rg)), ops.plan.counts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gradient_pass_matches_global(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    n, deg, ld = 6000, 6.0, 26
    pc = mp.spawn(_worker, args=(world, _free_port(), n, deg, ld, q), nprocs=world, join=False)
    res = [q.get(timeout=600) for _ in range(world)]
    while not pc.join():
        pass
    for rank, err, axe, gg, gg_ref, crr, crr_ref, counts in res:
        assert err <= 1e-13, (rank, err)
        assert axe <= 1e-12
        assert abs(gg - gg_ref) <= 1e-10 * gg_ref      # all-reduced scalars equal the global ones
        assert abs(crr - crr_ref) <= 1e-10 * (1 + abs(crr_ref))
        assert sum(counts) > 0                          # random graph: rows really cross blocks


def _solve_worker(rank, world, port, case, q, cfg_over=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2407_15049_b200 import driver, shard
        from paper_2407_15049_b200.device import Device
        from tests._golden import cfg_of, load, problem_from
        z = load(f"solve_{case}.npz")
        p = problem_from(z)
        cfg = dict(cfg_of(z))
        cfg.update(cfg_over or {})
        try:
            rep = shard.solve_sharded(p, driver.SolverConfig(**cfg), dev=Device())
        except Exception:
            import traceback
            q.put((rank, "error", traceback.format_exc(), None, None, None, None, None))
            raise
        tr = np.array([r[2:7] for r in rep.trace_rows], dtype=float).reshape(-1, 5)
        q.put((rank, rep.status, rep.objective, rep.err1, rep.err3, rep.err2, tr, rep.rank_history))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [("g1_like", 2), ("triangle_l2", 2), ("maxcut_2k_deg6", 3)])
def test_sharded_solve_within_reference_envelope(case, world):
    """A row-sharded solve (2-3 ranks) stays inside the reference's envelope, like the 1-GPU solve."""
    from tests._golden import load
    from tests.test_gpu_solve import first_dev
    z = load(f"solve_{case}.npz")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    # read the queue before joining: a child blocks on exit until its queued payload is consumed
    pc = mp.spawn(_solve_worker, args=(world, _free_port(), case, q), nprocs=world, join=False)
    res = []
    for _ in range(world):
        res.append(q.get(timeout=600))
        if res[-1][1] == "error":
            pytest.fail(f"rank {res[-1][0]} raised:\n{res[-1][2]}")
    res.sort(key=lambda t: t[0])
    while not pc.join():
        pass
    # every rank took the same decisions and reports the same numbers
    for r in res[1:]:
        assert r[1] == res[0][1] and r[2] == res[0][2] and np.array_equal(r[6], res[0][6])
    _, status, obj, err1, err3, err2, tr, ranks = res[0]
    ref = z["trace"]
    statuses = set(z["ulp_status"].tolist()) | {str(z["status"])}
    objs = np.append(z["ulp_objective"], float(z["objective"]))
    horizon = first_dev(tr, ref)
    print(f"{case} x{world}: status {status} obj {obj!r} rows {len(tr)} (ref {len(ref)}) horizon {horizon} "
          f"(ulp {int(z['ulp_horizon'].min())})")
    assert status in statuses
    assert horizon >= min(len(ref), len(tr), max(1, int(z["ulp_horizon"].min()) // 2))
    pad = 1e-6 * max(1.0, abs(objs).max())
    if status == "optimal":
        assert objs.min() - pad <= obj <= objs.max() + pad
    else:
        # capped, non-converged run (max_reopts=0, step cap): the final iterate lies far past
        # the chaotic horizon and a 5-run envelope under-samples it -- a sanity bound only
        spread = objs.max() - objs.min()
        assert objs.min() - 2 * spread <= obj <= objs.max() + 2 * spread


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_completion_follows_single_gpu_solve(world):
    """Non-diagonal constraints (matrix completion's symmetric pairs): constraint rows
    spread over the ranks, positions and multipliers through halos. A capped solve
    follows the 1-GPU solve's trace to 1e-9 (collectives staged through gloo here are
    slow, so the run is short)."""
    from paper_2407_15049_b200 import driver
    from tests._golden import cfg_of, load, problem_from
    from tests.test_gpu_solve import first_dev
    over = dict(admm_step_cap=40, max_reopts=0)
    z = load("solve_completion_30.npz")
    cfg = dict(cfg_of(z))
    cfg.update(over)
    single = driver.solve(problem_from(z), driver.SolverConfig(**cfg))
    ref = np.array([r[2:7] for r in single.trace_rows], dtype=float)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pc = mp.spawn(_solve_worker, args=(world, _free_port(), "completion_30", q, over), nprocs=world, join=False)
    res = []
    for _ in range(world):
        res.append(q.get(timeout=600))
        if res[-1][1] == "error":
            pytest.fail(f"rank {res[-1][0]} raised:\n{res[-1][2]}")
    res.sort(key=lambda t: t[0])
    while not pc.join():
        pass
    tr = res[0][6]
    for r in res[1:]:
        assert np.array_equal(r[6], tr)
    horizon = first_dev(tr, ref)
    print(f"completion_30 x{world}: rows {len(tr)} (1 GPU {len(ref)}) 1e-9 horizon {horizon}")
    assert horizon >= min(len(ref), len(tr), 300)
    # the capped run stops before convergence, past the chaotic horizon: a sanity bound only
    assert abs(res[0][2] - single.objective) <= 1e-3 * abs(single.objective)


def _reject_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2407_15049_b200 import shard
        from paper_2407_15049_b200.device import Device
        from tests._golden import load, problem_from
        try:
            shard.build_sharded_operators(problem_from(load("solve_random_sdp.npz")), rank, world, Device())
            q.put((rank, "built"))
        except NotImplementedError as e:
            q.put((rank, "rejected: " + str(e)))
    finally:
        dist.destroy_process_group()


def test_sharding_rejects_constraints_spanning_remote_rows():
    """Dense random constraints with positions touching no owned row: a clear error, no hang."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pc = mp.spawn(_reject_worker, args=(2, _free_port(), q), nprocs=2, join=False)
    res = [q.get(timeout=300) for _ in range(2)]
    while not pc.join():
        pass
    assert all(r[1].startswith("rejected") for r in res)


def _reorder_worker(rank, world, port, q, over):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2407_15049_b200 import driver, graphs, problem, reorder, shard
        from paper_2407_15049_b200.device import Device
        p = problem.build_maxcut(graphs.delaunay_like(900, seed=3))
        try:
            rep = shard.solve_sharded(p, driver.SolverConfig(reorder=True, **over), dev=Device())
            # halo of the C pattern with and without the locality order
            halo = []
            for prob in (p, reorder.permute(p, reorder.locality_order(p))[0]):
                dev = Device()
                dev.world, dev.group = world, None
                ops = shard.build_sharded_operators(prob, rank, world, dev, None)
                halo.append(ops.c_mat.cpat.halo.halo_bytes(2))
        except Exception:
            import traceback
            q.put((rank, "error", traceback.format_exc(), None, None, None))
            raise
        tr = np.array([r[2:7] for r in rep.trace_rows], dtype=float).reshape(-1, 5)
        q.put((rank, rep.status, rep.objective, tr, halo, rep.perm is not None))
    finally:
        dist.destroy_process_group()


def test_sharded_locality_ordered_solve():
    """SolverConfig(reorder=True) in the row-sharded solve: the mesh is relabelled in the
    locality order on every rank before the rows are split, so each rank's halo shrinks to
    the band at its block boundaries; the capped solve follows the 1-GPU reordered solve."""
    from paper_2407_15049_b200 import admm, alm, driver, graphs, problem, spectral
    from tests.test_gpu_solve import first_dev
    over = dict(admm_step_cap=60, max_reopts=0)
    p = problem.build_maxcut(graphs.delaunay_like(900, seed=3))
    # the sharded solve runs the multi-launch kernels: compare with those on one GPU
    admm.FUSED = alm.FUSED = spectral.FUSED = False
    try:
        single = driver.solve(p, driver.SolverConfig(reorder=True, **over))
    finally:
        admm.FUSED = alm.FUSED = spectral.FUSED = True
    ref = np.array([r[2:7] for r in single.trace_rows], dtype=float)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pc = mp.spawn(_reorder_worker, args=(world, _free_port(), q, over), nprocs=world, join=False)
    res = []
    for _ in range(world):
        res.append(q.get(timeout=600))
        if res[-1][1] == "error":
            pytest.fail(f"rank {res[-1][0]} raised:\n{res[-1][2]}")
    res.sort(key=lambda t: t[0])
    while not pc.join():
        pass
    tr = res[0][3]
    for r in res[1:]:
        assert np.array_equal(r[3], tr) and r[2] == res[0][2]
    for r in res:
        assert r[5]                                   # the order was applied
        assert r[4][1] * 4 <= r[4][0]                 # halo at least 4x smaller with the order
    horizon = first_dev(tr, ref)
    print(f"reordered mesh x{world}: rows {len(tr)} (1 GPU {len(ref)}) 1e-9 horizon {horizon}, "
          f"halo bytes {res[0][4][0]} -> {res[0][4][1]}")
    # the ALM stage and the first ADMM steps agree to 1e-9; later rows part by chaos
    assert horizon >= min(len(ref), len(tr), 100)
    assert abs(res[0][2] - single.objective) <= 1e-3 * abs(single.objective)


def _native_twin_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2407_15049_b200 import admm, alm, driver, shard
        from paper_2407_15049_b200.device import Device
        from tests._golden import cfg_of, load, problem_from
        z = load("solve_g1_like.npz")
        cfg = dict(cfg_of(z))
        cfg.update(admm_step_cap=60, max_reopts=1)
        p = problem_from(z)
        out = []
        for native in (True, False):
            alm.NATIVE = admm.NATIVE = native
            rep = shard.solve_sharded(p, driver.SolverConfig(**cfg), dev=Device())
            out.append((np.array([r[2:7] for r in rep.trace_rows], dtype=float), rep.objective, rep.gpu_launches))
        q.put((rank, out))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


def test_sharded_native_loops_match_python_twins():
    """Row-sharded solves run the native C++ ALM inner loop and ADMM step with the
    distributed hooks (halo exchange + rank-ordered slab reduction as callbacks,
    include/culorads.h cl_dist_hooks): bit-identical trace to the Python-driven loops."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    pc = mp.spawn(_native_twin_worker, args=(world, _free_port(), q), nprocs=world, join=False)
    res = [q.get(timeout=900) for _ in range(world)]
    while not pc.join():
        pass
    for rank, out in res:
        assert not isinstance(out, str), out
        (tn, on, ln), (tp, op, lp) = out
        print(f"rank {rank}: rows {len(tn)} objective {on!r} launches native {ln} python {lp}")
        assert len(tn) == len(tp) and np.array_equal(tn, tp) and on == op
