"""Multi-GPU P2P over Morton-range partitions.

One process per GPU.  Every rank builds the plan for its partition from the
global point set (deterministic synthetic generation makes that free), owns a
contiguous Morton range of tiles -- its targets and the sources of its boxes
-- and receives, per apply, the weights of the halo sources it needs from the
other ranks.  The exchange is the caller's collective over a torch
ProcessGroup (NCCL over NVLink/NVSwitch on a B200 node); packing the send
buffer and assembling [owned | halo] weights run in the library's kernels.

    dp = DistributedP2P(src, tgt, level=12, group=None)   # default process group
    phi_local = dp.apply(q_owned)          # this rank's targets, plan order
    phi_all = dp.gather(phi_local)         # allgatherv -> global plan order (every rank)
"""
from __future__ import annotations

import numpy as np

from . import p2p


class DistributedP2P:
    def __init__(self, src_xy=None, tgt_xy=None, *, group=None, device: int | None = None, host_staged: bool = False,
                 plan=None, **plan_kwargs):
        import torch
        import torch.distributed as dist
        self.dist, self.torch = dist, torch
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = (torch.cuda.current_device() if torch.cuda.is_available() else -1) if device is None else device
        self.host_staged = host_staged  # gloo / test mode: exchange through host tensors
        self.plan = plan if plan is not None else p2p.Plan(
            src_xy, tgt_xy, device=self.device, part_world=self.world, part_rank=self.rank, **plan_kwargs)
        self.src_ids = self.tgt_ids = None  # from_local: global ids of the received points
        info = self.plan.info
        self.info = info
        part = self.plan.export("partition").reshape(2, self.world + 1)
        self.src_begin, self.tgt_begin = part[0], part[1]
        hc = self.plan.export("halo_counts").reshape(2, self.world)
        self.recv_splits, self.send_splits = hc[0].tolist(), hc[1].tolist()
        dt = self.plan.torch_dtype
        if self.device >= 0:
            dev = torch.device("cuda", self.device)
            self._send = torch.empty(max(1, info["n_send"]), dtype=dt, device=dev)
            self._halo = torch.empty(max(1, info["n_halo"]), dtype=dt, device=dev)

    @classmethod
    def from_local(cls, src_xy, tgt_xy, src_ids, tgt_ids, *, level: int, group=None, device: int | None = None,
                   host_staged: bool = False, **plan_kwargs):
        """Each rank passes only the points it holds (any split of the global sets) with their
        global ids; no rank ever sees the global point set (north_star: "a one-time exchange
        distributes halo source points").  Collective:
          1. per-box counts of the held points (p2p_box_counts), summed over the ranks (allreduce);
          2. the partition from the global counts, and per held point the ranks that need it
             (p2p_partition_route: the owner of its box + the ranks whose tile regions hold it);
          3. one all-to-all of (x, y, id) records -- owned points and the halo sources;
          4. this rank's plan from what arrived (p2p_plan_create_local), identical to the plan
             the global builder makes for this rank.
        Weights then go in per owned source, in the order owned_source_ids() gives."""
        import torch
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        src_xy = np.ascontiguousarray(src_xy, dtype=np.float64).reshape(-1, 2)
        tgt_xy = np.ascontiguousarray(tgt_xy, dtype=np.float64).reshape(-1, 2)
        src_ids = np.ascontiguousarray(src_ids, dtype=np.int64)
        tgt_ids = np.ascontiguousarray(tgt_ids, dtype=np.int64)
        if device is None:
            device = torch.cuda.current_device() if torch.cuda.is_available() else -1
        on_dev = not host_staged and device >= 0 and dist.get_backend(group) == "nccl"
        cdev = torch.device("cuda", device) if on_dev else torch.device("cpu")
        # 1. global per-box counts
        counts = np.concatenate([p2p.p2p_box_counts(level, src_xy), p2p.p2p_box_counts(level, tgt_xy)])
        ct = torch.from_numpy(counts).to(cdev)
        dist.all_reduce(ct, group=group)
        counts = ct.cpu().numpy()
        B = len(counts) // 2
        cs, ctg = counts[:B], counts[B:]
        # 2. routing
        kw = dict(plan_kwargs)
        desc = p2p.make_desc(src_xy, tgt_xy, level=level, part_world=world, part_rank=rank, device=device, **kw)
        smask, tmask = p2p.p2p_partition_route(desc, src_ids, tgt_ids, cs, ctg)

        # 3. one all-to-all per point set: (x, y, id) records (ids < 2^53 are exact in float64)
        def route(xy, ids, mask):
            recs, cnt = [], []
            for r in range(world):
                sel = (mask >> np.uint32(r)) & np.uint32(1) == 1
                recs.append(np.column_stack([xy[sel], ids[sel].astype(np.float64)]))
                cnt.append(int(sel.sum()))
            send = torch.from_numpy(np.ascontiguousarray(np.concatenate(recs).reshape(-1))).to(cdev)
            sc = torch.tensor(cnt, dtype=torch.int64, device=cdev)
            rc = torch.empty_like(sc)
            dist.all_to_all_single(rc, sc, group=group)
            rcn = rc.cpu().tolist()
            recv = torch.empty(3 * sum(rcn), dtype=torch.float64, device=cdev)
            dist.all_to_all_single(recv, send, [3 * c for c in rcn], [3 * c for c in cnt], group=group)
            a = recv.cpu().numpy().reshape(-1, 3)
            return np.ascontiguousarray(a[:, :2]), a[:, 2].astype(np.int64)

        rs_xy, rs_id = route(src_xy, src_ids, smask)
        rt_xy, rt_id = route(tgt_xy, tgt_ids, tmask)
        # 4. this rank's plan
        plan = p2p.Plan(rs_xy, rt_xy, level=level, part_world=world, part_rank=rank, device=device, build="local",
                        local=(rs_id, rt_id, cs, ctg), **kw)
        self = cls(group=group, device=device, host_staged=host_staged, plan=plan)
        self.src_ids, self.tgt_ids = rs_id, rt_id
        self.src_xy_local, self.tgt_xy_local = rs_xy, rt_xy  # what arrived (the plan copied it)
        return self

    def owned_source_ids(self) -> np.ndarray:
        """from_local plans: global ids of this rank's owned sources, in the order apply() takes
        their weights (global plan order)."""
        gidx = self.plan.export("src_global")
        lo, hi = self.owned_source_range()
        return self.src_ids[self.plan.export("src_perm")[(gidx >= lo) & (gidx < hi)]]

    def target_ids(self) -> np.ndarray:
        """from_local plans: global ids of this rank's targets, in the order apply() returns them."""
        return self.tgt_ids[self.plan.export("tgt_perm")]

    @property
    def n_src_owned(self) -> int:
        return int(self.info["n_src_owned"])

    @property
    def n_tgt_local(self) -> int:
        return int(self.info["n_tgt_local"])

    def owned_source_range(self) -> tuple[int, int]:
        """Global plan-order range of the sources this rank owns."""
        return int(self.src_begin[self.rank]), int(self.src_begin[self.rank + 1])

    def exchange(self, q_owned, stream=None):
        """Halo weight exchange (a6): pack what the peers need, all-to-all, return the halo buffer.
        ``stream`` (a raw cudaStream_t handle): the pack kernel and the collective both run on it
        (torch collectives use the current stream, so it is made current for the call), so an
        apply enqueued on the same stream is ordered after the exchange."""
        torch = self.torch
        if stream is not None and stream != torch.cuda.current_stream(self.device).cuda_stream:
            with torch.cuda.stream(torch.cuda.ExternalStream(stream, device=torch.device("cuda", self.device))):
                return self._exchange(q_owned, stream)
        return self._exchange(q_owned, stream)

    def _exchange(self, q_owned, stream):
        info = self.info
        n_send, n_halo = int(info["n_send"]), int(info["n_halo"])
        if n_send:
            self.plan.halo_pack(q_owned, self._send, stream)
        send, halo = self._send[:n_send], self._halo[:n_halo]
        rs, ss = self.recv_splits, self.send_splits
        if send.is_complex():  # complex weights (Helmholtz) move as (re, im) float pairs
            send, halo = self.torch.view_as_real(send).reshape(-1), self.torch.view_as_real(halo).reshape(-1)
            rs, ss = [2 * x for x in rs], [2 * x for x in ss]
        if self.host_staged:
            recv = self.torch.empty(halo.numel(), dtype=halo.dtype)
            self.dist.all_to_all_single(recv, send.cpu(), rs, ss, group=self.group)
            halo.copy_(recv)
        else:
            self.dist.all_to_all_single(halo, send, rs, ss, group=self.group)
        return self._halo

    def exchange_async(self, q_owned, comm_stream, after=None):
        """Start the halo exchange on ``comm_stream`` (a torch.cuda.Stream) and return an event
        the compute stream can wait on: independent problems overlap one's exchange with
        another's kernel (bench.py's step).  ``after``: a stream whose queued work (the previous
        apply still reading the halo buffer) the exchange must follow."""
        torch = self.torch
        if after is not None:
            comm_stream.wait_stream(after)
        with torch.cuda.stream(comm_stream):
            self.exchange(q_owned, comm_stream.cuda_stream)
            ev = torch.cuda.Event()
            ev.record(comm_stream)
        return ev

    def apply(self, q_owned, out=None, *, accumulate: bool = False, stream=None, halo_ready=None):
        """phi for this rank's targets (plan order) from its owned weights (plan order).
        ``halo_ready``: an event from exchange_async (the exchange is then not repeated); the
        interior tiles run before waiting on it, so the exchange overlaps them."""
        torch = self.torch
        if out is None:
            out = torch.empty(max(1, self.n_tgt_local), dtype=self.plan.torch_dtype,
                              device=torch.device("cuda", self.device))
        if halo_ready is None:
            halo = self.exchange(q_owned, stream)
            self.plan.apply_dist(q_owned, halo, out, accumulate=accumulate, stream=stream)
            return out
        self.plan.apply_dist_interior(q_owned, out, accumulate=accumulate, stream=stream)
        cur = torch.cuda.current_stream(self.device) if stream is None else torch.cuda.ExternalStream(stream)
        cur.wait_event(halo_ready)
        self.plan.apply_dist_boundary(self._halo, out, accumulate=accumulate, stream=stream)
        return out

    def apply_overlapped(self, q_owned, comm_stream, out=None, *, accumulate: bool = False, stream=None):
        """One problem with its exchange overlapped: exchange on ``comm_stream`` while the
        interior tiles run on ``stream``; the boundary tiles wait for the halo."""
        torch = self.torch
        cur = torch.cuda.current_stream(self.device) if stream is None else torch.cuda.ExternalStream(stream)
        ev = self.exchange_async(q_owned, comm_stream, after=cur)
        return self.apply(q_owned, out, accumulate=accumulate, stream=stream, halo_ready=ev)

    # ---- peer-memory halo (SURVEY.md §8(e) alternative; p2p_apply_dist_peer): the halo weights
    # are read straight from the owners' buffers -- NVLink P2P loads on a B200 node -- by one
    # gather kernel, instead of pack + all_to_all + scatter.
    def enable_peer(self):
        """Allocate this rank's shared owned-weight buffer and map every peer's (CUDA IPC)."""
        torch = self.torch
        self._qpeer = torch.zeros(max(1, self.n_src_owned), dtype=self.plan.torch_dtype,
                                  device=torch.device("cuda", self.device))
        mine = p2p.p2p_ipc_export(self._qpeer.data_ptr())
        allh = [None] * self.world
        self.dist.all_gather_object(allh, mine, group=self.group)
        self._peers = [(0, 0) if r == self.rank else (p2p.p2p_ipc_open(allh[r][0], allh[r][1], self.device), allh[r][1])
                       for r in range(self.world)]

    def apply_peer(self, q_owned, out=None, *, accumulate: bool = False, stream=None):
        """phi for this rank's targets with the peer-memory halo.  Protocol: publish q_owned in
        the shared buffer, barrier (every rank's weights are in place), gather + apply, barrier
        (no rank overwrites its buffer while a peer may still read it)."""
        torch = self.torch
        if not hasattr(self, "_peers"):
            self.enable_peer()
        n = self.n_src_owned
        if n:
            self._qpeer[:n].copy_(q_owned[:n])
        torch.cuda.synchronize(self.device)
        self.dist.barrier(group=self.group)
        if out is None:
            out = torch.empty(max(1, self.n_tgt_local), dtype=self.plan.torch_dtype,
                              device=torch.device("cuda", self.device))
        s = stream or torch.cuda.current_stream(self.device).cuda_stream
        p2p.p2p_apply_dist_peer(self.plan.handle, self._qpeer.data_ptr() if n else 0, [p for p, _ in self._peers],
                                out.data_ptr(), int(accumulate), s)
        torch.cuda.synchronize(self.device)
        self.dist.barrier(group=self.group)
        return out

    def gather_peer(self, phi_local):
        """allgatherv (a11) over peer memory: every rank copies every shard straight from its
        owner's buffer (CUDA IPC mappings; NVLink reads on a node) -- no collective."""
        torch = self.torch
        dev = torch.device("cuda", self.device)
        if not hasattr(self, "_out_peers"):
            self._outbuf = torch.zeros(max(1, self.n_tgt_local), dtype=self.plan.torch_dtype, device=dev)
            mine = p2p.p2p_ipc_export(self._outbuf.data_ptr())
            allh = [None] * self.world
            self.dist.all_gather_object(allh, mine, group=self.group)
            self._out_peers = [(self._outbuf.data_ptr(), 0) if r == self.rank else
                               (p2p.p2p_ipc_open(allh[r][0], allh[r][1], self.device), allh[r][1])
                               for r in range(self.world)]
        n = self.n_tgt_local
        if n:
            self._outbuf[:n].copy_(phi_local[:n])
        torch.cuda.synchronize(self.device)
        self.dist.barrier(group=self.group)
        out = torch.empty(int(self.tgt_begin[-1]), dtype=self.plan.torch_dtype, device=dev)
        p2p.p2p_gather_peer(self.plan.handle, [p for p, _ in self._out_peers], out.data_ptr(),
                            torch.cuda.current_stream(self.device).cuda_stream)
        torch.cuda.synchronize(self.device)
        self.dist.barrier(group=self.group)
        return out

    # ---- device-synchronised peer exchange (p2p_apply_peer_sync / p2p_gather): the halo and the
    # result allgatherv as one-sided NVLink reads ordered by signal words in device memory -- no
    # host barrier per apply; the host only sets the mappings up once.
    def enable_sync(self):
        """Map every rank's published buffers and signal block (CUDA IPC), once."""
        if getattr(self, "_sync", None):
            return
        pw, po, sg = p2p.p2p_peer_buffers(self.plan.handle)
        mine = (p2p.p2p_ipc_export(pw), p2p.p2p_ipc_export(po), p2p.p2p_ipc_export(sg), self.send_splits)
        allh = [None] * self.world
        self.dist.all_gather_object(allh, mine, group=self.group)
        maps, ptrs = [], [[], [], []]
        for r in range(self.world):
            for k, own in enumerate((pw, po, sg)):
                if r == self.rank:
                    ptrs[k].append(own)
                else:
                    h, off = allh[r][k]
                    p = p2p.p2p_ipc_open(h, off, self.device)
                    maps.append((p, off))
                    ptrs[k].append(p)
        # my segment's offset in each owner's send buffer: its send entries for ranks before me
        displ = [int(sum(allh[o][3][:self.rank])) for o in range(self.world)]
        p2p.p2p_peer_connect(self.plan.handle, ptrs[0], ptrs[1], ptrs[2], displ)
        self._sync = maps

    def apply_sync(self, q_owned, out=None, *, accumulate: bool = False, stream=None):
        """phi for this rank's targets (plan order); the halo pulled from the owners' memory with
        device-side signalling (every rank calls it the same number of times)."""
        torch = self.torch
        self.enable_sync()
        if out is None:
            out = torch.empty(max(1, self.n_tgt_local), dtype=self.plan.torch_dtype,
                              device=torch.device("cuda", self.device))
        s = stream or torch.cuda.current_stream(self.device).cuda_stream
        p2p.p2p_apply_peer_sync(self.plan.handle, q_owned.data_ptr() if self.n_src_owned else 0, out.data_ptr(),
                                int(accumulate), s)
        return out

    def gather_sync(self, phi_local, out=None, stream=None):
        """allgatherv (a11) through the C ABI's p2p_gather: every rank's shard read from its
        owner's memory, device-synchronised (collective)."""
        torch = self.torch
        self.enable_sync()
        if out is None:
            out = torch.empty(max(1, int(self.tgt_begin[-1])), dtype=self.plan.torch_dtype,
                              device=torch.device("cuda", self.device))
        s = stream or torch.cuda.current_stream(self.device).cuda_stream
        p2p.p2p_gather(self.plan.handle, phi_local.data_ptr() if self.n_tgt_local else 0, out.data_ptr(), s)
        return out

    def check(self):
        """Raise if a device-side wait for a peer timed out (host-synchronous)."""
        p2p.p2p_peer_check(self.plan.handle)

    def gather(self, phi_local):
        """allgatherv (a11): every rank receives phi for all targets in global plan order."""
        torch = self.torch
        counts = np.diff(self.tgt_begin).astype(np.int64)
        cmax = int(counts.max()) if len(counts) else 0
        pad = torch.zeros(max(1, cmax), dtype=phi_local.dtype, device=phi_local.device)
        pad[: self.n_tgt_local].copy_(phi_local[: self.n_tgt_local])
        if pad.is_complex():  # collectives on the (re, im) float view
            real = torch.view_as_real(pad).reshape(-1)
            if self.host_staged:
                pr = [torch.empty_like(real, device="cpu") for _ in range(self.world)]
                self.dist.all_gather(pr, real.cpu(), group=self.group)
            else:
                pr = [torch.empty_like(real) for _ in range(self.world)]
                self.dist.all_gather(pr, real, group=self.group)
            parts = [torch.view_as_complex(p.reshape(-1, 2).contiguous()) for p in pr]
            return torch.cat([p[: int(c)].to(phi_local.device) for p, c in zip(parts, counts)])
        if self.host_staged:
            parts = [torch.empty_like(pad, device="cpu") for _ in range(self.world)]
            self.dist.all_gather(parts, pad.cpu(), group=self.group)
        else:
            parts = [torch.empty_like(pad) for _ in range(self.world)]
            self.dist.all_gather(parts, pad, group=self.group)
        return torch.cat([p[: int(c)].to(phi_local.device) for p, c in zip(parts, counts)])

    def close(self):
        for ptr, off in getattr(self, "_sync", None) or []:
            p2p.p2p_ipc_close(ptr, off)
        self._sync = None
        for ptr, off in getattr(self, "_peers", []):
            if ptr:
                p2p.p2p_ipc_close(ptr, off)
        self._peers = []
        for r, (ptr, off) in enumerate(getattr(self, "_out_peers", [])):
            if ptr and r != self.rank:
                p2p.p2p_ipc_close(ptr, off)
        self._out_peers = []
        self.plan.close()
