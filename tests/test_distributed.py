"""Multi-GPU host logic on CPU: two processes over gloo run paper_2204_10402_b200.distributed
with stand-in expander/solver functions (no GPU here), checking the partitioning, the node
accounting, the PVC found-flag cancel and the MVC bound exchange through the mailbox."""
import ctypes as C
import os
import socket
import time

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

N = 7  # vertices of the fake graph: a seed record is [cc, edges, deg[7]]


class FakeGraph:
    num_vertices = N


def fake_expander(graph, mode, k, target, device=0, stream=None):
    seeds = np.zeros((target + 3, 2 + N), np.uint32)
    seeds[:, 0] = np.arange(target + 3)  # tag = record index
    return dict(seeds=seeds, nodes=100, levels=5, best=9 if mode == "mvc" else k,
                greedy_size=9, found=False, cover=list(range(9)) if mode == "mvc" else [],
                kernel_launches=5)


def words_at(address):
    return np.ctypeslib.as_array((C.c_uint32 * 4).from_address(address))


def make_solver(rank, scenario, log):
    def solver(graph, seeds, mailbox, device, stream, initial_best=None, **kw):
        w = words_at(mailbox)
        log["tags"] = sorted(int(t) for t in seeds[:, 0])
        res = dict(status="complete", size=0, feasible=False, cover=[], worker_nodes=[len(seeds)],
                   nodes_total=10 * len(seeds), device_ms=1.0, kernel_launches=2,
                   cover_from_search=False)
        if scenario == "pvc_yes":
            if rank == 1:
                time.sleep(0.05)
                w[2], w[3] = 3, 1  # the device found a cover of size 3 <= k
                res.update(feasible=True, size=3, cover=[0, 1, 2])
            else:
                t0 = time.time()
                while not w[1]:  # wait for the monitor to forward the remote found flag
                    assert time.time() - t0 < 20, "cancel never arrived"
                    time.sleep(0.001)
                log["cancelled"] = True
        elif scenario == "mvc":
            log["initial_best"] = initial_best
            if rank == 0:
                time.sleep(0.05)
                w[2] = 5  # the device improved the bound to 5
                res.update(size=5, cover=[1, 2, 3, 4, 5], cover_from_search=True, feasible=True)
            else:
                t0 = time.time()
                while w[0] != 5:  # external bound delivered into this rank's mailbox
                    assert time.time() - t0 < 20, "bound never arrived"
                    time.sleep(0.001)
                log["ext_best"] = int(w[0])
                res.update(size=9, feasible=True)
        return res
    return solver


def worker(rank, world, port, scenario, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2204_10402_b200.distributed import Mailbox, solve_distributed
    log = {}
    mode, k = ("mvc", 0) if scenario == "mvc" else ("pvc", 4)
    r = solve_distributed(FakeGraph(), mode, k, frontier_per_rank=5, expander=fake_expander,
                          solver=make_solver(rank, scenario, log), mailbox=Mailbox(pinned=False),
                          period=0.001)
    out.put((rank, r, log))
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run(scenario, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=worker, args=(r, world, port, scenario, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        rank, r, log = q.get(timeout=120)
        res[rank] = (r, log)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_pvc_no_partition_and_node_accounting():
    res = run("pvc_no")
    target = 5 * 2 + 3  # expander returns target + 3 records
    tags0 = res[0][1]["tags"]
    tags1 = res[1][1]["tags"]
    assert tags0 == list(range(0, target, 2)) and tags1 == list(range(1, target, 2))
    for rank in (0, 1):
        r = res[rank][0]
        assert not r["feasible"] and r["status"] == "complete"
        assert r["nodes_total"] == 100 + 10 * target  # frontier once + every shard once
        assert r["rank_nodes"] == [10 * len(tags0), 10 * len(tags1)]


def test_pvc_found_flag_cancels_the_other_rank():
    res = run("pvc_yes")
    assert res[0][1].get("cancelled")
    for rank in (0, 1):
        r = res[rank][0]
        assert r["feasible"] and r["size"] == 3 and r["cover"] == [0, 1, 2]


def test_mvc_bound_is_exchanged_and_minimum_wins():
    res = run("mvc")
    assert res[1][1]["ext_best"] == 5
    assert res[0][1]["initial_best"] == 9
    for rank in (0, 1):
        r = res[rank][0]
        assert r["size"] == 5 and r["cover"] == [1, 2, 3, 4, 5]


def decided_expander(graph, mode, k, target, device=0, stream=None):
    """The frontier expansion itself found a cover (PVC decided, or the MVC optimum)."""
    seeds = np.zeros((0, 2 + N), np.uint32)
    return dict(seeds=seeds, nodes=7, levels=2, best=3 if mode == "mvc" else k, greedy_size=5,
                found=True, cover=[0, 2, 4], kernel_launches=2)


def worker_decided(rank, world, port, mode, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2204_10402_b200.distributed import Mailbox, solve_distributed
    calls = []

    def solver(graph, **kw):
        calls.append(1)
        raise AssertionError("no share to search")

    r = solve_distributed(FakeGraph(), mode, 4 if mode == "pvc" else 0, frontier_per_rank=5,
                          expander=decided_expander, solver=solver,
                          mailbox=Mailbox(pinned=False), period=0.001)
    out.put((rank, r, {"calls": len(calls)}))
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["pvc", "mvc"])
def test_frontier_decides_without_search_on_three_ranks(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=worker_decided, args=(r, 3, port, mode, q)) for r in range(3)]
    for p in ps:
        p.start()
    got = [q.get(timeout=120) for _ in range(3)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, r, log in got:
        assert log["calls"] == 0
        assert r["feasible"] and r["size"] == 3 and r["cover"] == [0, 2, 4]
        assert r["nodes_total"] == 7


# ---- exchange="peer": the IPC-handle rendezvous and the combination, with a stand-in shard --

class FakeShard:
    """Records what solve_distributed asks of a shards.Shard (no device)."""
    log = None

    def __init__(self, graph, mode, k, *, seeds=None, device=0, with_root=False, **kw):
        self.seeds = seeds
        self.kw = kw
        self.with_root = with_root
        self.rank = None
        FakeShard.log["opened"] = dict(n=0 if seeds is None else len(seeds), kw=sorted(kw),
                                       with_root=with_root)

    @property
    def work_units(self):
        return len(self.seeds) if self.seeds is not None else int(self.with_root)

    def export(self):
        return bytes([dist.get_rank()]) * 8

    def link_ipc(self, world, rank, handles, units):
        FakeShard.log["link"] = dict(world=world, rank=rank, handles=handles, units=list(units))

    def launch(self):
        FakeShard.log["launched"] = FakeShard.log.get("launched", 0) + 1

    def reset(self):
        FakeShard.log["resets"] = FakeShard.log.get("resets", 0) + 1

    def wait(self):
        n = self.work_units
        return dict(size=0, feasible=False, cover=[], cover_from_search=False, status="complete",
                    worker_nodes=[n], nodes_total=10 * n, device_ms=1.0, donated=n,
                    donated_peer=1, kernel_launches=2)

    def close(self):
        FakeShard.log["closed"] = True


def worker_peer(rank, world, port, out, fpr=2):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2204_10402_b200.distributed import solve_distributed
    FakeShard.log = {}
    r = solve_distributed(FakeGraph(), "pvc", 4, frontier_per_rank=fpr, expander=fake_expander,
                          shard_factory=FakeShard, exchange="peer", timeout_s=5)
    out.put((rank, r, FakeShard.log))
    dist.destroy_process_group()


def test_peer_exchange_rendezvous_on_three_ranks():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=worker_peer, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = {}
    for _ in range(world):
        rank, r, log = q.get(timeout=120)
        got[rank] = (r, log)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    total = 2 * world + 3  # fake_expander: target + 3 seed records, dealt i % world
    shares = [len(range(rk, total, world)) for rk in range(world)]
    for rank, (r, log) in got.items():
        assert log["opened"]["n"] == shares[rank] and log["opened"]["kw"] == ["timeout_s"]
        assert not log["opened"]["with_root"]
        assert log["link"]["world"] == world and log["link"]["rank"] == rank
        assert log["link"]["handles"] == [bytes([q]) * 8 for q in range(world)]  # rank order
        assert log["link"]["units"] == shares
        assert log["launched"] and log["closed"]
        assert r["exchange"] == "peer" and not r["feasible"] and r["status"] == "complete"
        assert r["nodes_total"] == 100 + 10 * total
        assert r["rank_nodes"] == [10 * n for n in shares]
        assert r["rank_donated_peer"] == [1] * world


def test_peer_exchange_root_only_start():
    """frontier_per_rank=0: no expansion; rank 0 starts from the root, the others empty (the
    linked worklists spread the work)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=worker_peer, args=(r, world, port, q, 0)) for r in range(world)]
    for p in ps:
        p.start()
    got = {}
    for _ in range(world):
        rank, r, log = q.get(timeout=120)
        got[rank] = (r, log)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, (r, log) in got.items():
        assert log["opened"]["n"] == 0 and log["opened"]["with_root"] == (rank == 0)
        assert log["link"]["units"] == [1, 0]
        assert r["frontier_nodes"] == 0 and r["nodes_total"] == 10


def worker_persistent(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2204_10402_b200.distributed import PeerSolver
    FakeShard.log = {}
    ps = PeerSolver(FakeGraph(), "pvc", 4, None, shard_factory=FakeShard)
    rs = [ps.solve() for _ in range(3)]
    ps.close()
    out.put((rank, rs, dict(FakeShard.log)))
    dist.destroy_process_group()


def test_peer_solver_links_once_and_resets_between_solves():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=worker_persistent, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = {}
    for _ in range(world):
        rank, rs, log = q.get(timeout=120)
        got[rank] = (rs, log)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, (rs, log) in got.items():
        assert log["launched"] == 3 and log["resets"] == 2 and log["closed"]
        assert log["link"]["units"] == [1, 0]  # linked once (the log keeps the one call)
        assert all(r["nodes_total"] == 10 and r["exchange"] == "peer" for r in rs)
