"""One process per GPU: a learner group whose synchronisation runs in libds
kernels that read and write the peers' buffers over NVLink P2P.

torch.distributed is only the plumbing (rendezvous and the one-time exchange
of CUDA IPC handles); the per-step traffic is

  SSGD       ds_shard_step : canonical-order reduce-scatter of the gradients
             + /world + momentum SGD on the owned chunks + all-gather of theta
             and its bf16 snapshot (RingAllreduceGroup.allreduce + sgd_step,
             collective.py:122-163, engines/ssgd.py:84-87)
  Hybrid     ds_shard_step mode 1 (weight average, engines/hybrid.py:97-99)
  ADPSGD     ds_pair_mix : (theta_i + theta_j) / 2 into both learners, each
             side mixing half the vector (adpsgd_mix, engines/adpsgd.py:36-43)
  H-ADPSGD   ds_shard_step inside a group + ds_pair_mix between member r of
             two groups

SSGD steps are bracketed by ds_peer_barrier device barriers on IPC-shared
flag words.  ADPSGD follows the reference's asynchronous protocol
(engines/adpsgd.py:115-288) as one-sided device work: the sender initiates
after its own update (exchange_async: lock the receiver's weights, mix over
NVLink on a comm stream, unlock), its next gradient overlaps the exchange
and only its next update waits for the ack (ack_gate); a receiver never
waits for anybody — its update takes its own weight lock (locked_update),
which is what makes the mix atomic against it (:280-285).  A slow learner
therefore delays only the exchanges that involve it, never a whole ring
(PAPER.md:252).  The partner schedule is the reference's Topology
(engines/common.py:38-75).  NCCL is the comparison transport only.
"""

from __future__ import annotations

import ctypes

from . import _lib
from .schedule import SENDER, Topology

_HB = 64  # DS_IPC_HANDLE_BYTES


def _arr(ptrs, ctype=ctypes.c_void_p):
    return (ctype * len(ptrs))(*ptrs)


def export_handle(dev_ptr: int) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle, byte offset) of the allocation holding dev_ptr."""
    lib = _lib.load()
    buf = (ctypes.c_uint8 * _HB)()
    off = ctypes.c_int64()
    _lib.check(lib.ds_ipc_export(ctypes.c_void_p(dev_ptr), buf, ctypes.byref(off)), "ds_ipc_export")
    return bytes(buf), int(off.value)


def adpsgd_partner(rank: int, world: int, iteration: int) -> int:
    """0-based partner of `rank` at (1-based) `iteration` under the
    reference's ring Topology: odd ids send, even ids receive; a sender's
    partner alternates right (odd iteration) / left (even iteration)
    (engines/common.py:64-69).  Receivers are the senders' partners."""
    topo = Topology(world)
    me = rank + 1
    if topo.role(me) == SENDER:
        return topo.partner(me, iteration) - 1
    for s in range(1, world + 1, 2):
        if topo.partner(s, iteration) == me:
            return s - 1
    raise ValueError(f"learner {me} has no sender at iteration {iteration}")  # pragma: no cover


def hadpsgd_layout(rank: int, groups: int, group_size: int) -> tuple[int, int]:
    """(group id, member index) of a rank: groups are contiguous rank blocks."""
    if rank < 0 or rank >= groups * group_size:
        raise ValueError("rank outside the group layout")
    return rank // group_size, rank % group_size


class PeerGroup:
    """The P2P view of one learner (a `blstm.Learner`) in a process group.

    Construction exchanges IPC handles of every learner's theta, gradient,
    bf16 snapshot and barrier-flag words (collective, all ranks), and maps
    the peers' buffers into this process."""

    def __init__(self, learner, rank: int, world: int, pg=None, timeout_s: float = 60.0):
        import torch
        import torch.distributed as dist

        if world < 1 or world > 16:
            raise ValueError("P2P groups hold 1..16 learners")
        self.L = learner
        self.rank, self.world = rank, world
        self.timeout_s = float(timeout_s)
        self.P = learner.obj.param_dim
        lib = _lib.load()
        dev = learner.theta.device
        self.flags = torch.zeros(64, dtype=torch.int32, device=dev)  # [writer rank] -> pair epoch
        # ctl[0]: lock word of this learner's weights (ds_peer_lock); the rest spare
        self.ctl = torch.zeros(16, dtype=torch.int32, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.pair_epochs = torch.zeros(64, dtype=torch.int32, device=dev)  # barriers shared with each rank
        self.comm = torch.cuda.Stream(device=dev)  # ADPSGD exchanges (overlap the next gradient)
        self.upd_ev = torch.cuda.Event()
        self.mix_ev = torch.cuda.Event()
        self.mix_pending = False
        snap = lib.ds_blstm_snapshot_ptr(learner.handle)
        mine = {
            "theta": export_handle(learner.theta.data_ptr()),
            "grad": export_handle(learner.grad.data_ptr()),
            "snap": export_handle(snap),
            "flags": export_handle(self.flags.data_ptr()),
            "ctl": export_handle(self.ctl.data_ptr()),
        }
        torch.cuda.synchronize(dev)  # buffers initialised before peers map them
        allh = [None] * world
        if world > 1:
            dist.all_gather_object(allh, mine, group=pg)
        else:
            allh = [mine]
        self._opened = []
        self.ptrs = {k: [0] * world for k in mine}
        local = {"theta": learner.theta.data_ptr(), "grad": learner.grad.data_ptr(), "snap": snap,
                 "flags": self.flags.data_ptr(), "ctl": self.ctl.data_ptr()}
        for r in range(world):
            for k in mine:
                if r == rank:
                    self.ptrs[k][r] = local[k]
                    continue
                h, off = allh[r][k]
                base = ctypes.c_void_p()
                p = ctypes.c_void_p()
                _lib.check(lib.ds_ipc_open(h, off, ctypes.byref(base), ctypes.byref(p)), "ds_ipc_open")
                self._opened.append(base.value)
                self.ptrs[k][r] = p.value
        if world > 1:
            dist.barrier(group=pg)

    # -- primitives -------------------------------------------------------------
    def barrier(self, members: list[int] | None = None) -> None:
        """Device barrier among `members` (world ranks, default all), ordered
        on the learner's stream."""
        members = list(range(self.world)) if members is None else list(members)
        lib = _lib.load()
        fl = _arr([self.ptrs["flags"][m] for m in members])
        rk = _arr(members, ctypes.c_int32)
        _lib.check(lib.ds_peer_barrier(len(members), fl, rk, self.rank, self.flags.data_ptr(),
                                       self.pair_epochs.data_ptr(), self.err.data_ptr(), self.timeout_s,
                                       self.L.stream.cuda_stream), "ds_peer_barrier")

    def attach_fused_ssgd(self, members: list[int] | None = None, chunk_count: int | None = None,
                          divisor: float = 0.0, max_blocks: int = 0) -> None:
        """Make L.train_step an SSGD group step: every layer's gradient block
        is reduced (canonical order), averaged, stepped and all-gathered into
        the members on the side stream as soon as it is final, overlapping
        the BPTT of the layers below (ds_blstm_set_group).  Bit-identical to
        gradient + ssgd_step; detach with detach_fused_ssgd()."""
        members = list(range(self.world)) if members is None else list(members)
        if self.rank not in members:
            raise ValueError("this rank is not a member of the group")
        if len(members) > _lib.DS_MAX_GROUP:
            raise ValueError("at most 16 members")
        d = _lib.DsGroupDesc()
        d.n = len(members)
        d.me = members.index(self.rank)
        d.my_rank = self.rank
        d.nchunks = chunk_count or len(members)
        d.divisor = float(divisor)
        d.max_blocks = int(max_blocks)
        for i, m in enumerate(members):
            d.ranks[i] = m
            d.thetas[i] = self.ptrs["theta"][m]
            d.grads[i] = self.ptrs["grad"][m]
            d.snaps[i] = self.ptrs["snap"][m]
            d.flags[i] = self.ptrs["flags"][m]
        d.own_flags = self.flags.data_ptr()
        d.pair_epochs = self.pair_epochs.data_ptr()
        d.err = self.err.data_ptr()
        d.timeout_s = self.timeout_s
        _lib.check(_lib.load().ds_blstm_set_group(self.L.handle, ctypes.byref(d)), "ds_blstm_set_group")

    def detach_fused_ssgd(self) -> None:
        _lib.check(_lib.load().ds_blstm_set_group(self.L.handle, None), "ds_blstm_set_group")

    def check(self) -> None:
        self.L.stream.synchronize()
        self.comm.synchronize()
        e = int(self.err.item())
        if e & 1:
            raise _lib.DsError("peer barrier timed out: a learner of the group stopped")
        if e & 2:
            raise _lib.DsError("peer weight lock timed out: a learner of the group stopped")

    # -- asynchronous ADPSGD (engines/adpsgd.py:115-288 as one-sided device work) ----
    def _lock(self, rank: int, stream) -> None:
        _lib.check(_lib.load().ds_peer_lock(self.ptrs["ctl"][rank], self.rank + 1, self.err.data_ptr(),
                                            self.timeout_s, stream.cuda_stream), "ds_peer_lock")

    def _unlock(self, rank: int, stream) -> None:
        _lib.check(_lib.load().ds_peer_unlock(self.ptrs["ctl"][rank], stream.cuda_stream), "ds_peer_unlock")

    def ack_gate(self) -> None:
        """Sender: the next update waits for the previous exchange's ack
        (engines/adpsgd.py:139-141) — a stream wait, the host never blocks."""
        if self.mix_pending:
            self.L.stream.wait_event(self.mix_ev)
            self.mix_pending = False

    def locked_update(self, lr: float) -> None:
        """Receiver: sgd_step under the learner's own lock, so an incoming mix
        lands entirely before or after it (the atomic region of
        engines/adpsgd.py:280-285)."""
        self._lock(self.rank, self.L.stream)
        self.L.sgd_step(lr)
        self._unlock(self.rank, self.L.stream)

    def exchange_async(self, peer: int) -> None:
        """Sender, after its update: adpsgd_mix with the receiver `peer` on the
        comm stream — lock the receiver's weights, (theta_i' + theta_j) / 2 into
        both learners over NVLink, unlock.  The sender's next gradient (on its
        pre-mix snapshot) overlaps it; only its next update waits (ack_gate)."""
        if peer == self.rank:
            raise ValueError("a learner cannot mix with itself")
        self.upd_ev.record(self.L.stream)
        self.comm.wait_event(self.upd_ev)
        self._lock(peer, self.comm)
        _lib.check(_lib.load().ds_pair_mix(self.L.theta.data_ptr(), self.ptrs["theta"][peer], None, None, self.P, -1,
                                           self.comm.cuda_stream), "ds_pair_mix")
        self._unlock(peer, self.comm)
        self.mix_ev.record(self.comm)
        self.mix_pending = True

    def update_exchange_async(self, peer: int, lr: float) -> None:
        """Sender, N1 fused variant: sgd_step + adpsgd_mix in one pass
        (ds_update_mix) on the comm stream under the receiver's lock.  The
        next gradient needs the refreshed snapshot, so the learner stream
        waits for it (no overlap of the exchange with the next gradient)."""
        lib = _lib.load()
        self.upd_ev.record(self.L.stream)
        self.comm.wait_event(self.upd_ev)
        self._lock(peer, self.comm)
        _lib.check(lib.ds_update_mix(self.L.theta.data_ptr(), self.L.vel.data_ptr(), self.L.grad.data_ptr(),
                                     self.ptrs["theta"][peer], lib.ds_blstm_snapshot_ptr(self.L.handle), float(lr),
                                     float(self.L.mu), self.P, self.L.flag.data_ptr(), self.comm.cuda_stream),
                   "ds_update_mix")
        self._unlock(peer, self.comm)
        self.mix_ev.record(self.comm)
        self.L.stream.wait_event(self.mix_ev)
        self.mix_pending = False
        self._refresh_aux()

    def _refresh_aux(self) -> None:
        lib = _lib.load()
        _lib.check(lib.ds_blstm_snapshot_aux(self.L.handle, self.L.theta.data_ptr(), self.L.stream.cuda_stream),
                   "ds_blstm_snapshot_aux")

    # -- strategies ---------------------------------------------------------------
    def ssgd_step(self, lr: float, members: list[int] | None = None, chunk_count: int | None = None,
                  divisor: float = 0.0, locked: bool = False) -> None:
        """One SSGD synchronisation of the member group (default: everyone):
        barrier -> owned-chunk reduce + SGD + all-gather -> barrier.
        locked=True (an H-ADPSGD receiver group): every member holds its own
        weight lock across the step, so no cross-group mix lands inside it."""
        members = list(range(self.world)) if members is None else list(members)
        w = len(members)
        me = members.index(self.rank)
        lib = _lib.load()
        if locked:
            self._lock(self.rank, self.L.stream)
        self.barrier(members)
        _lib.check(lib.ds_shard_step(w, me, _arr([self.ptrs["grad"][m] for m in members]),
                                     _arr([self.ptrs["theta"][m] for m in members]),
                                     _arr([self.ptrs["snap"][m] for m in members]), self.L.vel.data_ptr(), self.P,
                                     chunk_count or w, float(lr), float(self.L.mu), 0, float(divisor),
                                     self.L.stream.cuda_stream), "ds_shard_step")
        self.barrier(members)
        if locked:
            self._unlock(self.rank, self.L.stream)
        self._refresh_aux()

    def average(self, members: list[int] | None = None, chunk_count: int | None = None) -> None:
        """Hybrid pull: theta <- canonical-order sum / world in every member."""
        members = list(range(self.world)) if members is None else list(members)
        w = len(members)
        me = members.index(self.rank)
        lib = _lib.load()
        self.barrier(members)
        _lib.check(lib.ds_shard_step(w, me, None, _arr([self.ptrs["theta"][m] for m in members]),
                                     _arr([self.ptrs["snap"][m] for m in members]), None, self.P,
                                     chunk_count or w, 1.0, 0.0, 1, 0.0, self.L.stream.cuda_stream), "ds_shard_step")
        self.barrier(members)
        self._refresh_aux()

    def mix(self, peer: int) -> None:
        """adpsgd_mix with world rank `peer`: barrier -> each side averages
        half of the vector into both learners -> barrier."""
        if peer == self.rank:
            raise ValueError("a learner cannot mix with itself")
        lib = _lib.load()
        pair = sorted((self.rank, peer))
        self.barrier(pair)
        half = pair.index(self.rank)
        _lib.check(lib.ds_pair_mix(self.L.theta.data_ptr(), self.ptrs["theta"][peer],
                                   lib.ds_blstm_snapshot_ptr(self.L.handle), self.ptrs["snap"][peer], self.P, half,
                                   self.L.stream.cuda_stream), "ds_pair_mix")
        self.barrier(pair)
        self._refresh_aux()

    def close(self) -> None:
        if not getattr(self, "_opened", None):
            return
        self.L.stream.synchronize()
        lib = _lib.load()
        for b in self._opened:
            lib.ds_ipc_close(ctypes.c_void_p(b))
        self._opened = []


__all__ = ["PeerGroup", "adpsgd_partner", "hadpsgd_layout", "export_handle"]
