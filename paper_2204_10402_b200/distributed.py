"""Multi-GPU hybrid traversal: one process per GPU.

Partitioning — the worklist is the natural shard. Every rank expands the top of the search tree
with the same deterministic, level-synchronous device expansion (``vcg_expand_frontier``) until
the frontier holds ``frontier_per_rank * world`` open nodes, then seeds its own device worklist
with the records ``i % world == rank``. Sub-trees are independent given (degree array, |S|,
|E|), so there is no data-path collective: each GPU runs the single-GPU
hybrid kernel on its share.

Coupling — only the MVC bound and the PVC found flag cross GPUs. A host monitor thread per
rank exchanges {best, found, done} over a CPU (gloo) group every ``period`` seconds and writes
what it learns into the rank's pinned mailbox, which the running kernel polls (worker 0 folds an
external bound in with atomicMin and turns a remote "found" into its cancel flag). The exchange
never touches the GPU, so it cannot queue behind the persistent kernel.

Every tree node is visited exactly once across ranks (frontier nodes once, on the expansion;
frontier sub-trees once, on their owner), so PVC no-instance node counts stay equal to the
reference's.
"""
from __future__ import annotations

import ctypes as C
import threading
import time

import numpy as np

from . import _native as _n

_lib = _n.lib


class Mailbox:
    """Four host words the kernel can read/write while it runs:
    [0] external best (in), [1] cancel request (in), [2] device best (out), [3] found (out).

    ``pinned=True`` allocates device-mapped pinned memory (vcg_mailbox_alloc) — required when a
    real kernel polls it. ``pinned=False`` is for host-only protocol tests with a stand-in
    solver."""

    def __init__(self, pinned=True):
        self._pinned = pinned
        if pinned:
            p = C.POINTER(C.c_uint32)()
            _n.check(_lib.vcg_mailbox_alloc(4, C.byref(p)))
            self._ptr = p
            self.words = np.ctypeslib.as_array(p, shape=(4,))
        else:
            self.words = np.zeros(4, np.uint32)
            self._ptr = self.words.ctypes.data_as(C.POINTER(C.c_uint32))

    @property
    def address(self):
        return C.cast(self._ptr, C.c_void_p).value

    def close(self):
        if self._pinned and self._ptr:
            _lib.vcg_mailbox_free(self._ptr)
            self._ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def expand_frontier(graph, mode, k, target, device=0, stream=None, initial_best=0, engine="auto"):
    """Deterministic device expansion (vcg_expand_frontier) → dict with ``seeds`` as an
    (count, 2 + n) uint32 array of [cover_count, edge_count, degrees...] records. Graphs beyond
    the dense engine (n > 1024, or engine "sparse") expand on the sparse engine, one CTA per
    node of a level."""
    from . import _ENGINES
    p = _n.Params()
    _lib.vcg_params_init(C.byref(p))
    p.engine = _ENGINES[engine]
    p.mode = _n.VCG_PVC if mode == "pvc" else _n.VCG_MVC
    p.k = k
    p.device = device
    p.initial_best = initial_best or 0
    if stream is not None:
        p.stream = C.c_void_p(int(stream))
    f = _n.Frontier()
    _n.check(_lib.vcg_expand_frontier(graph._h, C.byref(p), int(target), C.byref(f)))
    try:
        n = graph.num_vertices
        cnt = int(f.num_seeds)
        seeds = (np.ctypeslib.as_array(f.seeds, shape=(cnt * (2 + n),)).reshape(cnt, 2 + n).copy()
                 if cnt else np.zeros((0, 2 + n), np.uint32))
        return dict(seeds=seeds, nodes=int(f.nodes_visited), levels=int(f.levels),
                    best=int(f.best), greedy_size=int(f.greedy_size), found=bool(f.found),
                    cover=[int(f.cover[i]) for i in range(f.cover_len)],
                    kernel_launches=int(f.kernel_launches))
    finally:
        _lib.vcg_frontier_free(C.byref(f))


class _Monitor(threading.Thread):
    """Host-side exchange of {best, found, done} between ranks (see module docstring)."""

    def __init__(self, group, mailbox, pvc, initial_best, period):
        super().__init__(daemon=True)
        self.group = group
        self.mb = mailbox
        self.pvc = pvc
        self.best = initial_best
        self.period = period
        self.done = threading.Event()
        self.global_best = initial_best
        self.global_found = False
        self.rounds = 0
        self.error = None

    def run(self):
        import torch
        import torch.distributed as dist
        world = dist.get_world_size(self.group)
        try:
            while True:
                out_best = int(self.mb.words[2])
                mine = self.best if out_best == 0 else min(self.best, out_best)
                t = torch.tensor([mine, int(self.mb.words[3]), int(self.done.is_set())],
                                 dtype=torch.int64)
                got = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
                dist.all_gather(got, t, group=self.group)
                g = torch.stack(got)
                self.rounds += 1
                self.global_best = int(g[:, 0].min())
                self.global_found = bool(g[:, 1].max())
                if not self.pvc and self.global_best < mine:
                    self.mb.words[0] = self.global_best
                if self.pvc and self.global_found and not self.mb.words[3]:
                    self.mb.words[1] = 1
                if bool(g[:, 2].min()):
                    return
                time.sleep(self.period)
        except Exception as e:  # surfaced by solve_distributed
            self.error = e


def _empty_result(graph, pvc):
    return dict(status="complete", size=0, feasible=False, cover=[], worker_nodes=[],
                nodes_total=0, device_ms=0.0, wall_ms=0.0, kernel_launches=0,
                cover_from_search=False, greedy_size=0)


def solve_distributed(graph, mode="pvc", k=0, *, exchange_group=None, frontier_per_rank=1024,
                      device=0, stream=None, period=0.002, solver=None, expander=None,
                      mailbox=None, exchange="peer", shard_factory=None, **solve_kw):
    """One rank's part of a multi-GPU solve; every rank of ``exchange_group`` (a CPU/gloo
    process group; default: the world group) must call it. Returns the combined result
    (identical on every rank): size/feasible/cover, per-rank node counts and timings.

    ``exchange="peer"``: the ranks' device worklists are linked through CUDA IPC / NVLink P2P
    (``shards.Shard``) — work donation between GPUs, peer-atomic bound, shared termination; the
    CPU group only carries the IPC handles once. ``exchange="host"``: static shares, bound and
    found flag through the host monitor below."""
    import torch.distributed as dist
    if mode == "pvc" and k < 1:
        raise ValueError("pvc requires k >= 1")
    if exchange == "peer" and graph.num_vertices > 1024:
        exchange = "host"  # linked device worklists are dense-engine shards; large n: static shares
    if exchange == "peer" and solver is None:
        return _solve_peer(graph, mode, k, exchange_group, frontier_per_rank, device,
                           expander or expand_frontier, shard_factory, solve_kw)
    pvc = mode == "pvc"
    rank = dist.get_rank(exchange_group)
    world = dist.get_world_size(exchange_group)
    expander = expander or expand_frontier
    if solver is None:
        from . import solve_mvc, solve_pvc

        def solver(g, **kw):
            return (solve_pvc(g, k, raw=True, **kw) if pvc else solve_mvc(g, raw=True, **kw))

    t0 = time.perf_counter()
    fr = expander(graph, mode, k, frontier_per_rank * world, device=device, stream=stream,
                  **({"engine": solve_kw["engine"]} if "engine" in solve_kw else {}))
    share = fr["seeds"][rank::world]
    decided = pvc and fr["found"]
    res = _empty_result(graph, pvc)
    mb = mailbox or Mailbox()
    mon = _Monitor(exchange_group, mb, pvc, fr["best"], period)
    mon.start()
    try:
        if not decided and len(share):
            kw = dict(solve_kw, seeds=share, mailbox=mb.address, device=device, stream=stream)
            if not pvc:
                kw["initial_best"] = fr["best"]
            res = solver(graph, **kw)
    finally:
        mon.done.set()
        mon.join()
        if mailbox is None:
            mb.close()
    if mon.error is not None:
        raise mon.error
    wall_ms = (time.perf_counter() - t0) * 1e3

    # combine (every rank gets the same answer)
    mine = dict(size=res["size"], feasible=res["feasible"], cover=res["cover"],
                from_search=bool(res.get("cover_from_search")), status=res["status"],
                worker_nodes=res["worker_nodes"], nodes=res["nodes_total"],
                device_ms=res["device_ms"], wall_ms=wall_ms,
                launches=res.get("kernel_launches", 0))
    allr = [None] * world
    dist.all_gather_object(allr, mine, group=exchange_group)
    nodes = fr["nodes"] + sum(r["nodes"] for r in allr)
    if pvc:
        feasible = fr["found"] or any(r["feasible"] for r in allr)
        if fr["found"]:
            cover = fr["cover"]
        else:
            cover = next((r["cover"] for r in allr if r["feasible"]), [])
        size = len(cover) if feasible else 0
    else:
        feasible = True
        cands = [(len(fr["cover"]), fr["cover"])]
        cands += [(r["size"], r["cover"]) for r in allr if r["from_search"]]
        size, cover = min(cands, key=lambda c: c[0])
    statuses = [r["status"] for r in allr]
    status = next((s for s in statuses if s != "complete"), "complete")
    if pvc and feasible:
        status = "complete"
    return dict(size=size if feasible else None, feasible=feasible, cover=cover, status=status,
                nodes_total=nodes, frontier_nodes=fr["nodes"], frontier_levels=fr["levels"],
                frontier_size=int(len(fr["seeds"])),
                rank_nodes=[r["nodes"] for r in allr],
                rank_device_ms=[r["device_ms"] for r in allr],
                rank_wall_ms=[r["wall_ms"] for r in allr],
                worker_nodes=[w for r in allr for w in r["worker_nodes"]],
                kernel_launches=fr["kernel_launches"] + mine["launches"],
                exchange_rounds=mon.rounds, greedy_size=fr["greedy_size"])


class PeerSolver:
    """One rank's persistent shard for repeated multi-GPU solves of one (graph, mode, k): the
    shard is opened, its CUDA IPC handles exchanged over the CPU group and the peers mapped
    ONCE; every solve() then only resets the device state (all ranks reset before any launch),
    launches, waits, and gathers the small per-rank results. Rank 0 starts from the root (or
    from a deterministic frontier share, frontier_per_rank > 0)."""

    def __init__(self, graph, mode, k, group, *, device=0, frontier_per_rank=0, expander=None,
                 shard_factory=None, detail=True, **solve_kw):
        import torch.distributed as dist
        from .shards import Shard, combine, root_frontier
        self._combine = combine
        Shard = shard_factory or Shard
        self.graph, self.mode, self.k, self.group = graph, mode, k, group
        self.detail = detail  # gather every worker's node count (the report's worker_nodes)
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if frontier_per_rank:
            fr = (expander or expand_frontier)(graph, mode, k, frontier_per_rank * self.world,
                                               device=device)
            fr["frontier_size"] = int(len(fr["seeds"]))
        else:  # rank 0 starts from the root; donation between GPUs spreads the work
            fr = root_frontier(graph, mode, k)
        self.frontier = fr
        share = fr["seeds"][self.rank::self.world]
        self.decided = (mode == "pvc" and fr["found"]) or (frontier_per_rank and not len(fr["seeds"]))
        self.shard = None
        self.fresh = True
        if self.decided:
            return
        extra = {} if mode == "pvc" else {"initial_best": fr["best"]}
        self.shard = Shard(graph, mode, k, seeds=share if len(share) else None, device=device,
                           with_root=not frontier_per_rank and self.rank == 0, **extra,
                           **solve_kw)
        handles = [None] * self.world
        dist.all_gather_object(handles, self.shard.export(), group=group)
        units = [None] * self.world
        dist.all_gather_object(units, self.shard.work_units, group=group)
        self.shard.link_ipc(self.world, self.rank, handles, units)

    def solve(self):
        import torch.distributed as dist
        t0 = time.perf_counter()
        parts = []
        if self.shard is not None:
            if not self.fresh:
                self.shard.reset()
            self.fresh = False
            dist.barrier(group=self.group)  # every shard (re)initialised before any launch
            self.shard.launch()
            mine = self.shard.wait()
            # (the gather is also the barrier that keeps every kernel done before any reset)
            parts = self._gather(mine)
        out = self._combine(self.graph, self.mode, self.frontier, parts,
                            (time.perf_counter() - t0) * 1e3)
        out["exchange"] = "peer"
        return out

    _SCALARS = ("nodes_total", "feasible", "size", "cover_from_search", "donated",
                "donated_peer", "kernel_launches", "h2d_bytes", "d2h_bytes", "greedy_size")
    _STATUS = ("complete", "timeout", "budget")

    def _gather(self, mine):
        """Every rank's part: the scalars in one small tensor all-gather; covers (only when a
        rank has one to offer) and per-worker node counts (detail) as pickled objects."""
        import torch
        import torch.distributed as dist
        v = [int(mine.get(x, 0)) for x in self._SCALARS]
        v += [self._STATUS.index(mine["status"]) if mine["status"] in self._STATUS else 0,
              int(round(mine["device_ms"] * 1e6))]
        t = torch.tensor(v, dtype=torch.int64)
        got = [torch.zeros_like(t) for _ in range(self.world)]
        dist.all_gather(got, t, group=self.group)
        parts = []
        for g in got:
            g = g.tolist()
            d = dict(zip(self._SCALARS, g))
            d["feasible"] = bool(d["feasible"])
            d["cover_from_search"] = bool(d["cover_from_search"])
            d["status"] = self._STATUS[g[len(self._SCALARS)]]
            d["device_ms"] = g[len(self._SCALARS) + 1] / 1e6
            d["cover"], d["worker_nodes"] = [], []
            parts.append(d)
        need_cover = any(p["feasible"] if self.mode == "pvc" else p["cover_from_search"]
                         for p in parts)
        if need_cover or self.detail:
            extra = [None] * self.world
            dist.all_gather_object(
                extra, dict(cover=mine["cover"] if need_cover else [],
                            worker_nodes=mine["worker_nodes"] if self.detail else []),
                group=self.group)
            for p, e in zip(parts, extra):
                p.update(e)
        return parts

    def close(self):
        if self.shard is not None:
            self.shard.close()
            self.shard = None


def _solve_peer(graph, mode, k, group, frontier_per_rank, device, expander, shard_factory,
                solve_kw):
    """solve_distributed with device-linked worklists: a one-shot PeerSolver."""
    ps = PeerSolver(graph, mode, k, group, device=device, frontier_per_rank=frontier_per_rank,
                    expander=expander, shard_factory=shard_factory, **solve_kw)
    try:
        return ps.solve()
    finally:
        ps.close()
