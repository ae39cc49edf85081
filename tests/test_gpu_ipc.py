"""Multi-process shards linked through CUDA IPC (distributed.solve_distributed, exchange="peer"):
two processes on the one GPU of the test box. Their kernels are time-sliced rather than
co-resident, which is slow but exercises every step of the cross-process path: handle export /
open, the shard-activity count, donations into the other process's ring, cancel and bound
stores into its control block."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def worker(rank, world, port, mode, k, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2204_10402_b200 as vc
    from paper_2204_10402_b200.configs import load_config
    from paper_2204_10402_b200.distributed import solve_distributed
    g = load_config("c1")
    r = solve_distributed(g, mode, k, frontier_per_rank=64, device=0, exchange="peer",
                          timeout_s=120)
    ok = r["cover"] == [] or vc.verify_cover(g, r["cover"])
    out.put((rank, {x: r[x] for x in ("size", "feasible", "status", "nodes_total", "rank_nodes",
                                      "rank_donated_peer", "exchange")}, ok))
    dist.destroy_process_group()


def run(mode, k, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=worker, args=(r, world, port, mode, k, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = {}
    for _ in range(world):
        rank, r, ok = q.get(timeout=300)
        got[rank] = (r, ok)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


def test_ipc_shards_pvc_no_instance_exact(config_golden):
    gold = config_golden["c1"]
    got = run("pvc", gold["pvc_no_k"])
    for rank, (r, ok) in got.items():
        assert r["exchange"] == "peer" and r["status"] == "complete" and not r["feasible"]
        assert r["nodes_total"] == gold["pvc_no_nodes"], r


def test_ipc_shards_mvc_optimum(config_golden):
    gold = config_golden["c1"]
    got = run("mvc", 0)
    for rank, (r, ok) in got.items():
        assert r["status"] == "complete" and r["size"] == gold["mvc"] and ok, r
