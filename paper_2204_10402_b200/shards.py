"""Multi-shard solves with device-to-device work donation (include/vcgpu.h
``vcg_session_*``).

A shard is one dense-engine search with its own device worklist: one per GPU, or several
on one device. Linked shards exchange work and state through peer memory, with no host in
the loop and no collective:

* a worker whose peer shard is below its donation threshold writes its oldest stacked node
  straight into that shard's ring slot (NVLink P2P / CUDA IPC stores, then a system-scope
  release);
* an improved MVC bound reaches every shard by peer ``atomicMin``;
* a PVC "found", a timeout or a node budget cancels every shard;
* the solve ends when shard 0's count of shards with non-zero ``pending`` reaches zero.

This replaces the reference's one shared ``GlobalWorklist`` (worklist.cpp:11-48) across GPUs.

``solve_sharded`` runs all shards in this process: several devices, or several shards on
one device for tests. ``distributed.solve_distributed(exchange="peer")`` runs one shard per
process and exchanges CUDA IPC handles over the CPU process group.
"""
from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _native as _n

_lib = _n.lib


class Shard:
    """One ``vcg_session``: open (validate, greedy, buffers, seeds), link, launch, wait."""

    def __init__(self, graph, mode="pvc", k=0, *, seeds=None, with_root=False,
                 strategy="gpu", workers=0, capacity=4096, threshold_fraction=0.5,
                 timeout_s=None, node_budget=None, device=0, initial_best=0,
                 donate_oldest=None, engine="auto"):
        from . import _params
        if mode == "pvc" and k < 1:
            raise ValueError("pvc requires k >= 1")
        self.graph = graph
        self.mode = mode
        self.num_seeds = 0 if seeds is None else len(seeds)
        self.with_root = bool(with_root) and self.num_seeds == 0
        p, self._keep = _params(mode, k, strategy, workers, capacity, threshold_fraction, 8, 50,
                                timeout_s, node_budget, device=device, seeds=seeds,
                                initial_best=initial_best, donate_oldest=donate_oldest,
                                engine=engine)
        self._p = p
        h = C.c_void_p()
        _n.check(_lib.vcg_session_open(graph._h, C.byref(p), int(self.with_root), C.byref(h)))
        self._h = h

    @property
    def work_units(self):
        """Initial worklist entries (seeds, or 1 for the root)."""
        return self.num_seeds or int(self.with_root)

    def export(self) -> bytes:
        buf = (C.c_ubyte * _lib.vcg_session_handle_bytes())()
        _n.check(_lib.vcg_session_export(self._h, buf))
        return bytes(buf)

    def link_ipc(self, world, rank, handles, work_units):
        blob = b"".join(handles)
        units = np.ascontiguousarray(work_units, dtype=np.uint64)
        _n.check(_lib.vcg_session_link_ipc(self._h, world, rank, blob, units.ctypes.data))

    def launch(self):
        _n.check(_lib.vcg_session_launch(self._h))

    def reset(self):
        """Fresh search state for another solve (buffers, IPC mappings and links kept)."""
        _n.check(_lib.vcg_session_reset(self._h))

    def wait(self):
        from . import _result_dict
        r = _n.Result()
        _n.check(_lib.vcg_session_wait(self._h, C.byref(r)))
        try:
            out = _result_dict(r)
            out.pop("_worker_nodes_np", None)
            return out
        finally:
            _lib.vcg_result_free(C.byref(r))

    def close(self):
        if getattr(self, "_h", None):
            _lib.vcg_session_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def link_local(shards):
    arr = (C.c_void_p * len(shards))(*[s._h.value for s in shards])
    _n.check(_lib.vcg_session_link_local(arr, len(shards)))


def combine(graph, mode, frontier, parts, wall_ms):
    """The multi-shard answer from the frontier expansion and every shard's result.

    * PVC: feasible if any part found a cover.
    * MVC: the smallest certificate among the frontier's and the shards' search covers.

    Node counts add up: frontier nodes once, each shard its own sub-trees."""
    pvc = mode == "pvc"
    nodes = frontier["nodes"] + sum(r["nodes_total"] for r in parts)
    if pvc:
        feasible = frontier["found"] or any(r["feasible"] for r in parts)
        cover = frontier["cover"] if frontier["found"] else next(
            (r["cover"] for r in parts if r["feasible"]), [])
        size = len(cover) if feasible else None
    else:
        feasible = True
        cands = [(len(frontier["cover"]), frontier["cover"])]
        cands += [(r["size"], r["cover"]) for r in parts if r["cover_from_search"]]
        size, cover = min(cands, key=lambda c: c[0])
    statuses = [r["status"] for r in parts]
    status = next((s for s in statuses if s != "complete"), "complete")
    if pvc and feasible:
        status = "complete"
    return dict(size=size, feasible=feasible, cover=cover, status=status, nodes_total=nodes,
                frontier_nodes=frontier["nodes"], frontier_levels=frontier["levels"],
                frontier_size=frontier.get("frontier_size", 0),
                rank_nodes=[r["nodes_total"] for r in parts],
                rank_device_ms=[r["device_ms"] for r in parts],
                rank_donated=[r["donated"] for r in parts],
                rank_donated_peer=[r["donated_peer"] for r in parts],
                rank_idle_share=[r.get("timeline", {}).get("idle_share") for r in parts],
                worker_nodes=[w for r in parts for w in r["worker_nodes"]],
                kernel_launches=frontier["kernel_launches"] + sum(r["kernel_launches"] for r in parts),
                greedy_size=max([frontier["greedy_size"]] + [r.get("greedy_size", 0) for r in parts]),
                wall_ms=wall_ms,
                h2d_bytes=sum(r.get("h2d_bytes", 0) for r in parts),
                d2h_bytes=sum(r.get("d2h_bytes", 0) for r in parts))


def root_frontier(graph, mode, k):
    """No expansion: shard 0 starts from the root and device-to-device donation spreads the
    work (the greedy cover is the MVC certificate to beat, as in run_hybrid)."""
    from . import greedy_approx
    size, cover = greedy_approx(graph) if mode == "mvc" else (0, [])  # (PVC: the shards report it)
    return dict(seeds=np.zeros((0, 2 + graph.num_vertices), np.uint32), nodes=0, levels=0,
                best=size if mode == "mvc" else k, greedy_size=size, found=False,
                cover=[c + graph.id_base for c in cover] if mode == "mvc" else [],
                kernel_launches=0, frontier_size=0)


class ShardedSolver:
    """Persistent in-process shards (several devices, or several shards of one device): opened
    and linked once, then every solve() only resets the device state — the multi-shard setup
    cost (buffers, links) is paid once, not per solve. Root start (shard 0), donation spreads
    the work."""

    def __init__(self, graph, mode="pvc", k=0, *, devices=(0, 0), workers_per_shard=None, **kw):
        self.graph, self.mode, self.k = graph, mode, k
        self.frontier = root_frontier(graph, mode, k)
        if workers_per_shard is None:
            same = max(devices.count(d) for d in set(devices))
            workers_per_shard = 0 if same == 1 else device_workers(graph, devices[0]) // same
        extra = {} if mode == "pvc" else {"initial_best": self.frontier["best"]}
        self.shards = []
        try:
            for r, dev in enumerate(devices):
                self.shards.append(Shard(graph, mode, k, with_root=r == 0, device=dev,
                                         workers=workers_per_shard, **extra, **kw))
            link_local(self.shards)
        except Exception:
            self.close()
            raise
        self.fresh = True

    def solve(self):
        t0 = time.perf_counter()
        if not self.fresh:
            for s in self.shards:  # (all reset before any launches)
                s.reset()
        self.fresh = False
        for s in self.shards:
            s.launch()
        parts = [s.wait() for s in self.shards]
        return combine(self.graph, self.mode, self.frontier, parts,
                       (time.perf_counter() - t0) * 1e3)

    def close(self):
        for s in self.shards:
            s.close()
        self.shards = []


def solve_sharded(graph, mode="pvc", k=0, *, devices=(0, 0), frontier_per_shard=0,
                  workers_per_shard=None, skew=False, **kw):
    """All shards in this process, linked through device memory (peer access between GPUs).

    ``frontier_per_shard=0`` (default): shard 0 starts from the root, the others empty, and
    donation spreads the work. Otherwise the shards start from a deterministic frontier
    (``vcg_expand_frontier``, one launch per tree level) dealt round robin; ``skew=True`` deals
    it all to shard 0. Several shards on one device must share it: ``workers_per_shard``
    defaults to an equal split of the full-device worker count, so every shard stays resident
    at once."""
    from .distributed import expand_frontier
    world = len(devices)
    if world < 1:
        raise ValueError("need at least one shard")
    t0 = time.perf_counter()
    if frontier_per_shard:
        fr = expand_frontier(graph, mode, k, frontier_per_shard * world, device=devices[0])
        fr["frontier_size"] = int(len(fr["seeds"]))
    else:
        fr = root_frontier(graph, mode, k)
    decided = mode == "pvc" and fr["found"]
    if workers_per_shard is None:
        same = max(devices.count(d) for d in set(devices))
        workers_per_shard = 0 if same == 1 else device_workers(graph, devices[0]) // same
    shards, parts = [], []
    try:
        if not decided and (len(fr["seeds"]) or not frontier_per_shard):
            extra = {} if mode == "pvc" else {"initial_best": fr["best"]}
            for r, dev in enumerate(devices):
                share = (fr["seeds"] if r == 0 else fr["seeds"][:0]) if skew else fr["seeds"][r::world]
                shards.append(Shard(graph, mode, k, seeds=share if len(share) else None,
                                    with_root=not frontier_per_shard and r == 0,
                                    device=dev, workers=workers_per_shard, **extra, **kw))
            link_local(shards)
            for s in shards:
                s.launch()
            parts = [s.wait() for s in shards]
    finally:
        for s in shards:
            s.close()
    return combine(graph, mode, fr, parts, (time.perf_counter() - t0) * 1e3)


def device_workers(graph, device=0):
    """Workers (warps) of a full-device solve of ``graph``: shards on one device split them."""
    w = C.c_uint32()
    _n.check(_lib.vcg_device_workers(graph._h, device, C.byref(w)))
    return int(w.value)
