"""Run a row-sharded golden solve with W ranks on cuda:0 (gloo) and dump stacks if it hangs. Dev tool.

    python tools/shard_debug.py CASE WORLD
"""
import faulthandler
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch.multiprocessing as mp  # noqa: E402


def worker(rank, world, port, case):
    import torch
    import torch.distributed as dist
    faulthandler.dump_traceback_later(180, exit=True)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2407_15049_b200 import driver, shard
    from paper_2407_15049_b200.device import Device
    from tests._golden import cfg_of, load, problem_from
    z = load(f"solve_{case}.npz")
    p = problem_from(z)
    ops = shard.build_sharded_operators(p, rank, world, Device(), None)
    print(f"rank {rank}: rows {ops.row_range} cons {ops.con_range} m_own {ops.problem.m}", flush=True)
    rep = shard.solve_sharded(p, driver.SolverConfig(**cfg_of(z)), dev=Device())
    print(f"rank {rank}: {rep.status} {rep.objective!r} rows {len(rep.trace_rows)}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(worker, args=(int(sys.argv[2]), port, sys.argv[1]), nprocs=int(sys.argv[2]), join=True)
