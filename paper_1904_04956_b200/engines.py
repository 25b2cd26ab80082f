"""Learner engines — the reference strategy API (engines/*.py) driving device
learners.

Each engine keeps the reference's actor structure, channel wiring and
lock/counter bookkeeping (so a VirtualClock run produces the same draw /
update / exchange order, staleness samples, counts and byte totals as the
reference), while every weight-vector operation goes to the backend
(backend.GpuBackend: the sm_100a kernels; tests also plug a float64 numpy
backend).  Weights never leave the device inside the loop.

  run_single   engines/single.py:14-74     (the 1-GPU "SSGD batch 256" point)
  run_ssgd     engines/ssgd.py:28-141      (+ fused allreduce/SGD kernel, K11)
  run_adpsgd   engines/adpsgd.py:65-346    (+ pairwise mix kernel, K10)
  run_hadpsgd  SURVEY §8 a19: ADPSGD between groups, SSGD inside a group
  run_hybrid   engines/hybrid.py:25-174    (weight allreduce, staleness 1)

Snapshot rule (engines/adpsgd.py:132-134): the gradient of an update is
computed on the learner's weights as of its DRAW.  The device snapshot
(bf16 operand copy) is refreshed by the fused SGD kernel after every own
update; a DRAW re-casts it only if the weights were mutated since (a mix),
which reproduces the reference's `snap = st.weights.copy()` exactly.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np

from .metrics import MetricsRecord, StalenessRecord, staleness_summary
from .runtime import DelayModel, RunAborted, VirtualClock
from .schedule import Topology, MinibatchPool, epoch_minibatches, learning_rate, make_chunk_plan, static_partition


# ---------------------------------------------------------------------------
# errors / results / messages (engines/common.py:16-114)

class ChecksumError(RuntimeError):
    """A received weight payload failed integrity validation (torn snapshot)."""


class EngineFailure(RuntimeError):
    def __init__(self, epoch: int, cause: BaseException):
        super().__init__(f"epoch {epoch}: {cause}")
        self.epoch = epoch
        self.cause = cause


class EngineAborted(RuntimeError):
    def __init__(self, message: str, records: list):
        super().__init__(message)
        self.records = records


@dataclass
class RunResult:
    weights: np.ndarray
    records: list
    trace: dict = field(default_factory=dict)


@dataclass(frozen=True)
class WeightMessage:
    """Timestamped weight payload (common.py:78-104).  On the device path the
    payload is a reference to the sender's learner (the mix kernel reads it
    over NVLink/HBM), so no copy is shipped.  With `checksum=True` runs
    (debug mode) the message carries a 128-bit device digest of the weights
    it stands for (ds_digest) and `validate` recomputes it on the live
    buffer: a request proves the sender's weights were not touched between
    shipping and the receiver's mix (no torn snapshot), a reply proves both
    learners hold the identical mean.  Mismatch -> ChecksumError, as in the
    reference.  Without checksums ordering is structural (streams, locks)."""

    origin: int
    timestamp: int
    payload: object
    checksum: str = ""
    digest_fn: object = None

    @classmethod
    def snapshot(cls, origin: int, timestamp: int, payload, digest_fn=None) -> "WeightMessage":
        return cls(origin, timestamp, payload, digest_fn(payload) if digest_fn else "", digest_fn)

    def validate(self, against=None) -> None:
        if not self.checksum:
            return None
        live = self.digest_fn(self.payload if against is None else against)
        if live != self.checksum:
            raise ChecksumError(f"weights from learner {self.origin} (ts {self.timestamp}) changed in flight: "
                                f"{live} != {self.checksum}")


def _make_backend(objective, dataset, batch_size: int, backend):
    if backend is not None:
        return backend
    from .backend import GpuBackend

    return GpuBackend(objective, dataset, max_batch=batch_size)


def _check_epochs(epochs: int, schedule) -> None:
    if epochs < 0:
        raise ValueError(f"epochs must be >= 0, got {epochs}")
    if epochs > schedule.total_epochs:
        raise ValueError(f"epochs ({epochs}) exceeds schedule.total_epochs ({schedule.total_epochs})")


def _w0(objective, seed, init_weights):
    if init_weights is not None:
        return np.array(init_weights, dtype=np.float64, copy=True)
    return 0.1 * np.random.default_rng((seed, 0)).standard_normal(objective.param_dim)


def _frames(dataset, batch) -> int:
    x = getattr(dataset, "inputs", None)
    per = x.shape[1] if x is not None and x.ndim == 3 else 1
    return len(batch) * per


# ---------------------------------------------------------------------------
def run_single(objective, dataset, schedule, *, epochs: int, batch_size: int, seed: int, momentum: float = 0.9,
               delays: DelayModel | None = None, clock=None, init_weights=None, backend=None) -> RunResult:
    """Sequential minibatch SGD (engines/single.py:14-74) on one device learner."""
    _check_epochs(epochs, schedule)
    clock = clock or VirtualClock()
    delays = delays or DelayModel()
    be = _make_backend(objective, dataset, batch_size, backend)
    compute_delay = delays.compute_delay_fn(1)
    L = be.create(_w0(objective, seed, init_weights), momentum)
    records: list = []
    staleness = StalenessRecord("single")

    def body():
        for epoch in range(1, epochs + 1):
            try:
                batches = epoch_minibatches(dataset, batch_size, seed, epoch)
                t0 = clock.now()
                frames = 0
                for k, batch in enumerate(batches):
                    d = compute_delay()
                    if d > 0:
                        clock.sleep(d)
                    # gradient + sgd_step (single.py:53-55) as one fused device step
                    be.train_step(L, batch, learning_rate(schedule, epoch, k, len(batches)))
                    frames += _frames(dataset, batch)
                be.check(L)
                wall = clock.now() - t0
                records.append(MetricsRecord(epoch=epoch, heldout_loss=be.heldout_loss(L), epoch_wall_s=wall,
                                             minibatch_counts=[len(batches)], staleness_mean=0.0, staleness_max=0,
                                             bytes_exchanged=0, frames_per_s=frames / wall if wall > 0 else None))
            except RunAborted:
                raise
            except Exception as exc:
                raise EngineFailure(epoch, exc) from exc

    clock.run([body])
    return RunResult(weights=be.weights(L), records=records, trace={"staleness": staleness, "backend": be})


# ---------------------------------------------------------------------------
class DeviceRingGroup:
    """RingAllreduceGroup (collective.py:81-163) for device learners.

    The reference protocol — generation counters, 2(world-1) phases of
    per-chunk messages in canonical owner order, per-rank phase and byte
    counters — runs unchanged on the clock's channels, so simulated time and
    the byte accounting match the reference.  The data never moves through
    the channels: when the last rank of a generation enters, the fused
    reduce (+ /world + momentum SGD, or weight average) kernel is enqueued
    for every rank's owned chunks (K11).
    """

    def __init__(self, clock, plan, delay_fn_for_edge, backend, elem_bytes: int):
        self.plan = plan
        self.world = plan.world
        self._inbox = [clock.channel(delay_fn_for_edge(r) if delay_fn_for_edge else None) for r in range(self.world)]
        self._gen = [0] * self.world
        self.phases = [0] * self.world
        self.bytes_sent = [0] * self.world
        self._sizes = [hi - lo for lo, hi in plan.bounds]
        self._be = backend
        self._eb = elem_bytes
        self._arrived: dict = {}
        self._mu = threading.Lock()

    def reset_counters(self) -> None:
        self.phases = [0] * self.world
        self.bytes_sent = [0] * self.world

    def _send(self, rank, gen, phase, chunk):
        self._inbox[(rank + 1) % self.world].put((gen, phase, chunk))
        self.bytes_sent[rank] += self._sizes[chunk] * self._eb

    def _recv(self, rank, gen, phase, chunk):
        got = self._inbox[rank].get()
        if got != (gen, phase, chunk):
            raise RuntimeError(f"collective protocol violation at rank {rank}: expected "
                               f"(gen={gen}, phase={phase}, chunk={chunk}), got "
                               f"(gen={got[0]}, phase={got[1]}, chunk={got[2]})")

    def allreduce(self, rank: int, members: list, op) -> None:
        """Collective entry for `rank`; `op()` issues the device reduction and
        is run once per generation by the last rank to enter."""
        gen = self._gen[rank]
        self._gen[rank] += 1
        with self._mu:
            n = self._arrived.get(gen, 0) + 1
            self._arrived[gen] = n
            last = n == self.world
            if last:
                del self._arrived[gen]
        if last:
            op()
        w = self.world
        phase = 0
        for s in range(w - 1):
            for j in self.plan.chunks_of((rank - s) % w):
                self._send(rank, gen, phase, j)
            for j in self.plan.chunks_of((rank - s - 1) % w):
                self._recv(rank, gen, phase, j)
            self.phases[rank] += 1
            phase += 1
        for s in range(w - 1):
            for j in self.plan.chunks_of((rank + 1 - s) % w):
                self._send(rank, gen, phase, j)
            for j in self.plan.chunks_of((rank - s) % w):
                self._recv(rank, gen, phase, j)
            self.phases[rank] += 1
            phase += 1


def run_ssgd(objective, dataset, schedule, *, learners: int, epochs: int, batch_size: int, seed: int,
             momentum: float = 0.9, delays: DelayModel | None = None, clock=None, chunk_count: int | None = None,
             record_iterates: bool = False, init_weights=None, backend=None) -> RunResult:
    """Synchronous SGD (engines/ssgd.py:28-141): gradient -> canonical ring
    allreduce / lambda -> lr(k, q) -> momentum SGD, fused on the device."""
    if learners < 2:
        raise ValueError(f"ssgd needs at least 2 learners, got {learners}")
    _check_epochs(epochs, schedule)
    clock = clock or VirtualClock()
    delays = delays or DelayModel()
    be = _make_backend(objective, dataset, batch_size, backend)
    plan = make_chunk_plan(objective.param_dim, learners, chunk_count)
    group = DeviceRingGroup(clock, plan, delays.comm_delay_fn, be, be.elem_bytes)
    w0 = _w0(objective, seed, init_weights)
    L = {i: be.create(w0, momentum) for i in range(1, learners + 1)}
    members = [L[i] for i in range(1, learners + 1)]
    report_ch = clock.channel()
    go = {i: clock.channel() for i in range(1, learners + 1)}
    records: list = []
    staleness = StalenessRecord("ssgd")
    staleness_by_learner = {i: [] for i in range(1, learners + 1)}

    def learner(i: int):
        rank = i - 1
        compute_delay = delays.compute_delay_fn(i)

        def body():
            stagger = delays.initial_stagger(i)
            if stagger > 0:
                clock.sleep(stagger)
            for epoch in range(1, epochs + 1):
                try:
                    mine = static_partition(epoch_minibatches(dataset, batch_size, seed, epoch), learners)[rank]
                    samples = []
                    for k, batch in enumerate(mine):
                        d = compute_delay()
                        if d > 0:
                            clock.sleep(d)
                        be.gradient(L[i], batch)
                        lr = learning_rate(schedule, epoch, k, len(mine))
                        group.allreduce(rank, members, lambda lr=lr: be.group_step(members, lr, chunk_count))
                        samples.append(0)
                    if i == 1:
                        be.check(L[i])
                except RunAborted:
                    raise
                except Exception as exc:
                    raise EngineFailure(epoch, exc) from exc
                report_ch.put((i, len(mine), samples))
                go[i].get()

        return body

    def orchestrator():
        t0 = clock.now()
        for epoch in range(1, epochs + 1):
            reports = {}
            for _ in range(learners):
                i, count, samples = report_ch.get()
                reports[i] = (count, samples)
                staleness_by_learner[i].extend(samples)
            wall = clock.now() - t0
            all_samples = [s for i in sorted(reports) for s in reports[i][1]]
            staleness.samples.extend(all_samples)
            mean, mx = staleness_summary(all_samples)
            frames = sum(reports[i][0] for i in reports) * batch_size * getattr(objective, "frames", 1)
            records.append(MetricsRecord(epoch=epoch, heldout_loss=be.heldout_loss(L[1]), epoch_wall_s=wall,
                                         minibatch_counts=[reports[i][0] for i in sorted(reports)],
                                         staleness_mean=mean, staleness_max=mx,
                                         bytes_exchanged=sum(group.bytes_sent),
                                         frames_per_s=frames / wall if wall > 0 else None))
            group.reset_counters()
            for i in range(1, learners + 1):
                go[i].put(True)
            t0 = clock.now()

    clock.run([learner(i) for i in range(1, learners + 1)] + [orchestrator])
    return RunResult(weights=be.weights(L[1]), records=records,
                     trace={"staleness": staleness, "staleness_by_learner": staleness_by_learner, "backend": be})


# ---------------------------------------------------------------------------
@dataclass
class _State:
    dev: object
    lock: threading.Lock = field(default_factory=threading.Lock)
    iteration: int = 0
    mutations: int = 0
    snap_mut: int = 0   # mutation count the device snapshot reflects
    staleness: list = field(default_factory=list)
    exchanges: int = 0


class _Unit:
    """One ADPSGD learner: a single device learner (ADPSGD) or a group of
    identical members stepping synchronously (H-ADPSGD)."""

    def __init__(self, be, members: list, chunk_count=None):
        self.be = be
        self.members = members
        self.chunks = chunk_count

    def snapshot(self):
        for m in self.members:
            self.be.snapshot(m)

    def gradient(self, batch, dataset):
        if len(self.members) == 1:
            self.be.gradient(self.members[0], batch)
            return
        # contiguous slices of the drawn super-batch; each member's CE gradient
        # is scaled by 1/(frames of the whole batch) so the group sum is the
        # gradient of the union batch
        total = _frames(dataset, batch)
        for m, part in zip(self.members, np.array_split(np.asarray(batch), len(self.members))):
            if len(part) == 0:  # short final batch: this member contributes nothing
                self.be.zero_grad(m)
            else:
                self.be.gradient(m, part, frames_total=float(total))

    def update(self, lr):
        if len(self.members) == 1:
            self.be.sgd_step(self.members[0], lr)
        else:
            self.be.group_step(self.members, lr, self.chunks, divisor=1.0)

    def mix(self, other: "_Unit"):
        for a, b in zip(self.members, other.members):
            self.be.mix(a, b)

    def check(self):
        for m in self.members:
            self.be.check(m)


def _run_gossip(objective, dataset, schedule, *, units: int, epochs: int, batch_size: int, seed: int,
                momentum: float, delays, clock, record_trace: bool, init_weights, backend, group_size: int,
                chunk_count=None, strategy: str = "adpsgd", checksum: bool = False) -> RunResult:
    topo = Topology(units)
    _check_epochs(epochs, schedule)
    clock = clock or VirtualClock()
    delays = delays or DelayModel()
    be = _make_backend(objective, dataset, max(1, -(-batch_size // group_size)), backend)
    pool = MinibatchPool(epoch_minibatches(dataset, batch_size, seed, 1) if epochs else [], units)
    payload_bytes = objective.param_dim * be.elem_bytes * group_size
    w0 = _w0(objective, seed, init_weights)
    states = {i: _State(dev=_Unit(be, [be.create(w0, momentum) for _ in range(group_size)], chunk_count))
              for i in range(1, units + 1)}

    inbox = {j: clock.channel(delays.comm_delay_fn(j)) for j in topo.receivers()}
    reply = {i: clock.channel(delays.comm_delay_fn(i)) for i in topo.senders()}
    job = {i: clock.channel() for i in topo.senders()}
    ack = {i: clock.channel() for i in topo.senders()}
    quiesced = {j: clock.channel() for j in topo.receivers()}
    report_ch = clock.channel()
    go = {i: clock.channel() for i in range(1, units + 1)}
    records: list = []
    staleness = StalenessRecord(strategy)
    exchange_log: list = []
    staleness_by_learner = {i: [] for i in range(1, units + 1)}

    def unit_digest(unit: "_Unit") -> str:
        return "".join(be.digest(m) for m in unit.members)

    digest = unit_digest if checksum else None

    def draw_snapshot(st: _State):
        # caller holds st.lock: weights as of this DRAW (adpsgd.py:132-134)
        if st.snap_mut != st.mutations:
            st.dev.snapshot()
            st.snap_mut = st.mutations
        return st.mutations

    def local_update(st: _State, epoch, k, pool_size, mut0):
        lr = learning_rate(schedule, epoch, k, pool_size)
        st.staleness.append(st.mutations - mut0)
        st.dev.update(lr)  # fused SGD refreshes the snapshot
        st.mutations += 1
        st.snap_mut = st.mutations
        st.iteration += 1

    def sender_main(i: int):
        st = states[i]
        compute_delay = delays.compute_delay_fn(i)

        def body():
            stagger = delays.initial_stagger(i)
            if stagger > 0:
                clock.sleep(stagger)
            for epoch in range(1, epochs + 1):
                try:
                    pool_size = pool.size
                    pending = False
                    while True:
                        drawn = pool.next(i)
                        if drawn is None:
                            break
                        k, batch = drawn
                        with st.lock:
                            mut0 = draw_snapshot(st)
                        clock.sleep(compute_delay())
                        st.dev.gradient(batch, dataset)
                        if pending:
                            ack[i].get()
                            pending = False
                        with st.lock:
                            local_update(st, epoch, k, pool_size, mut0)
                            msg = WeightMessage.snapshot(i, st.iteration, st.dev, digest)
                            partner = topo.partner(i, st.iteration)
                        job[i].put(("exchange", msg, partner))
                        pending = True
                    if pending:
                        ack[i].get()
                    job[i].put(("epoch_done", None, None))
                    st.dev.check()
                except RunAborted:
                    raise
                except Exception as exc:
                    raise EngineFailure(epoch, exc) from exc
                with st.lock:
                    samples = st.staleness
                    st.staleness = []
                report_ch.put((i, samples, st.exchanges))
                st.exchanges = 0
                go[i].get()
            job[i].put(("stop", None, None))

        return body

    def sender_agent(i: int):
        st = states[i]

        def body():
            last_ts: dict = {}
            while True:
                kind, msg, partner = job[i].get()
                if kind == "stop":
                    return
                if kind == "epoch_done":
                    inbox[topo.left(i)].put(("epoch_done", i))
                    inbox[topo.right(i)].put(("epoch_done", i))
                    continue
                inbox[partner].put(("exchange", msg))
                resp: WeightMessage = reply[i].get()
                resp.validate(against=st.dev)  # the receiver wrote the identical mean into both
                if resp.timestamp < last_ts.get(resp.origin, -1):
                    raise RuntimeError(f"non-monotone timestamp from learner {resp.origin}: "
                                       f"{resp.timestamp} after {last_ts[resp.origin]}")
                last_ts[resp.origin] = resp.timestamp
                with st.lock:
                    # the device mean was written into both sides at the
                    # receiver's atomic reply+mix; this is the sender's SMIX
                    st.mutations += 1
                    st.exchanges += 1
                    if record_trace:
                        exchange_log.append((i, resp.origin))
                ack[i].put(True)

        return body

    def receiver_main(j: int):
        st = states[j]
        compute_delay = delays.compute_delay_fn(j)

        def body():
            stagger = delays.initial_stagger(j)
            if stagger > 0:
                clock.sleep(stagger)
            for epoch in range(1, epochs + 1):
                try:
                    pool_size = pool.size
                    while True:
                        drawn = pool.next(j)
                        if drawn is None:
                            break
                        k, batch = drawn
                        with st.lock:
                            mut0 = draw_snapshot(st)
                        clock.sleep(compute_delay())
                        st.dev.gradient(batch, dataset)
                        with st.lock:
                            local_update(st, epoch, k, pool_size, mut0)
                    quiesced[j].get()
                    st.dev.check()
                except RunAborted:
                    raise
                except Exception as exc:
                    raise EngineFailure(epoch, exc) from exc
                with st.lock:
                    samples = st.staleness
                    st.staleness = []
                exchanges = st.exchanges
                st.exchanges = 0
                report_ch.put((j, samples, exchanges))
                go[j].get()
            inbox[j].put(("stop", None))

        return body

    def receiver_agent(j: int):
        st = states[j]

        def body():
            markers = 0
            last_ts: dict = {}
            while True:
                item = inbox[j].get()
                if item[0] == "stop":
                    return
                if item[0] == "epoch_done":
                    markers += 1
                    if markers == 2:
                        markers = 0
                        quiesced[j].put(True)
                    continue
                msg: WeightMessage = item[1]
                msg.validate()
                if msg.timestamp < last_ts.get(msg.origin, -1):
                    raise RuntimeError(f"non-monotone timestamp from learner {msg.origin}: "
                                       f"{msg.timestamp} after {last_ts[msg.origin]}")
                last_ts[msg.origin] = msg.timestamp
                with st.lock:
                    st.dev.mix(msg.payload)  # identical mean into both sides (K10)
                    mine = WeightMessage.snapshot(j, st.iteration, st.dev, digest)
                    st.mutations += 1
                    st.exchanges += 1
                reply[msg.origin].put(mine)

        return body

    def orchestrator():
        t0 = clock.now()
        for epoch in range(1, epochs + 1):
            reports = {}
            for _ in range(units):
                i, samples, exchanges = report_ch.get()
                reports[i] = (samples, exchanges)
                staleness_by_learner[i].extend(samples)
            wall = clock.now() - t0
            counts = pool.counts.copy()
            members = [m for i in sorted(reports) for m in states[i].dev.members]
            avg = be.average(members)
            all_samples = [s for i in sorted(reports) for s in reports[i][0]]
            staleness.samples.extend(all_samples)
            mean, mx = staleness_summary(all_samples)
            n_exchanges = sum(reports[i][1] for i in topo.senders())
            frames = sum(counts) * batch_size * getattr(objective, "frames", 1)
            records.append(MetricsRecord(epoch=epoch, heldout_loss=be.heldout_loss(avg), epoch_wall_s=wall,
                                         minibatch_counts=counts, staleness_mean=mean, staleness_max=mx,
                                         bytes_exchanged=2 * n_exchanges * payload_bytes,
                                         frames_per_s=frames / wall if wall > 0 else None))
            if epoch < epochs:
                pool.reset(epoch_minibatches(dataset, batch_size, seed, epoch + 1))
            for i in range(1, units + 1):
                go[i].put(True)
            t0 = clock.now()

    actors = []
    for i in topo.senders():
        actors.append(sender_main(i))
        actors.append(sender_agent(i))
    for j in topo.receivers():
        actors.append(receiver_main(j))
        actors.append(receiver_agent(j))
    actors.append(orchestrator)
    clock.run(actors)

    all_members = [m for i in range(1, units + 1) for m in states[i].dev.members]
    weights = w0 if epochs == 0 else be.weights(be.average(all_members))
    trace = {"staleness": staleness, "staleness_by_learner": staleness_by_learner, "backend": be}
    if record_trace:
        trace["exchanges"] = exchange_log
    return RunResult(weights=weights, records=records, trace=trace)


def run_adpsgd(objective, dataset, schedule, *, learners: int, epochs: int, batch_size: int, seed: int,
               momentum: float = 0.9, delays: DelayModel | None = None, clock=None, record_trace: bool = False,
               init_weights=None, backend=None, checksum: bool = False) -> RunResult:
    """Asynchronous decentralized parallel SGD on the bipartite ring
    (engines/adpsgd.py:65-346); returns the uniform average of all learners.
    checksum=True validates every exchanged payload with a device digest
    (debug mode of the reference's WeightMessage checksum)."""
    return _run_gossip(objective, dataset, schedule, units=learners, epochs=epochs, batch_size=batch_size, seed=seed,
                       momentum=momentum, delays=delays, clock=clock, record_trace=record_trace,
                       init_weights=init_weights, backend=backend, group_size=1, checksum=checksum)


def run_hadpsgd(objective, dataset, schedule, *, groups: int, group_size: int, epochs: int, batch_size: int,
                seed: int, momentum: float = 0.9, delays: DelayModel | None = None, clock=None,
                record_trace: bool = False, init_weights=None, backend=None,
                chunk_count: int | None = None) -> RunResult:
    """Hierarchical ADPSGD: `groups` ADPSGD learners on the
    ring, each a group of `group_size` GPUs that split the drawn batch of
    group_size * batch_size sequences into contiguous slices and take one
    synchronous allreduce step (frame-weighted, fused SGD); member r of a
    group gossips with member r of the partner group.  Its schedule equals
    the reference run_adpsgd(learners=groups, batch_size=group_size*batch_size)."""
    if group_size < 1:
        raise ValueError(f"group_size must be >= 1, got {group_size}")
    return _run_gossip(objective, dataset, schedule, units=groups, epochs=epochs, batch_size=group_size * batch_size,
                       seed=seed, momentum=momentum, delays=delays, clock=clock, record_trace=record_trace,
                       init_weights=init_weights, backend=backend, group_size=group_size, chunk_count=chunk_count,
                       strategy="hadpsgd")


# ---------------------------------------------------------------------------
def run_hybrid(objective, dataset, schedule, *, learners: int, epochs: int, batch_size: int, seed: int,
               momentum: float = 0.9, delays: DelayModel | None = None, clock=None, chunk_count: int | None = None,
               record_iterates: bool = False, init_weights=None, backend=None) -> RunResult:
    """Paper Hybrid (engines/hybrid.py:25-174): pull the previous weight
    allreduce / lambda, gradient, local momentum SGD, push into the agent's
    allreduce; staleness 1 after the first iteration."""
    if learners < 2:
        raise ValueError(f"hybrid needs at least 2 learners, got {learners}")
    _check_epochs(epochs, schedule)
    clock = clock or VirtualClock()
    delays = delays or DelayModel()
    be = _make_backend(objective, dataset, batch_size, backend)
    plan = make_chunk_plan(objective.param_dim, learners, chunk_count)
    group = DeviceRingGroup(clock, plan, delays.comm_delay_fn, be, be.elem_bytes)
    w0 = _w0(objective, seed, init_weights)
    L = {i: be.create(w0, momentum) for i in range(1, learners + 1)}
    members = [L[i] for i in range(1, learners + 1)]
    push = {i: clock.channel() for i in range(1, learners + 1)}
    pull = {i: clock.channel() for i in range(1, learners + 1)}
    report_ch = clock.channel()
    go = {i: clock.channel() for i in range(1, learners + 1)}
    records: list = []
    staleness = StalenessRecord("hybrid")
    staleness_by_learner = {i: [] for i in range(1, learners + 1)}

    def learner(i: int):
        rank = i - 1
        compute_delay = delays.compute_delay_fn(i)

        def body():
            first = True
            pending = False
            stagger = delays.initial_stagger(i)
            if stagger > 0:
                clock.sleep(stagger)
            for epoch in range(1, epochs + 1):
                try:
                    mine = static_partition(epoch_minibatches(dataset, batch_size, seed, epoch), learners)[rank]
                    samples = []
                    for k, batch in enumerate(mine):
                        if pending:
                            pull[i].get()  # device weights already hold the consensus
                            pending = False
                        samples.append(0 if first else 1)
                        first = False
                        d = compute_delay()
                        if d > 0:
                            clock.sleep(d)
                        be.gradient(L[i], batch)
                        be.sgd_step(L[i], learning_rate(schedule, epoch, k, len(mine)))
                        push[i].put(True)
                        pending = True
                    pull[i].get()
                    pending = False
                    if i == 1:
                        be.check(L[i])
                except RunAborted:
                    raise
                except Exception as exc:
                    raise EngineFailure(epoch, exc) from exc
                report_ch.put((i, len(mine), samples))
                go[i].get()
            push[i].put(None)

        return body

    def agent(i: int):
        rank = i - 1

        def body():
            while True:
                item = push[i].get()
                if item is None:
                    return
                group.allreduce(rank, members, lambda: be.group_average(members, chunk_count))
                pull[i].put(True)

        return body

    def orchestrator():
        t0 = clock.now()
        for epoch in range(1, epochs + 1):
            reports = {}
            for _ in range(learners):
                i, count, samples = report_ch.get()
                reports[i] = (count, samples)
                staleness_by_learner[i].extend(samples)
            wall = clock.now() - t0
            all_samples = [s for i in sorted(reports) for s in reports[i][1]]
            staleness.samples.extend(all_samples)
            mean, mx = staleness_summary(all_samples)
            frames = sum(reports[i][0] for i in reports) * batch_size * getattr(objective, "frames", 1)
            records.append(MetricsRecord(epoch=epoch, heldout_loss=be.heldout_loss(L[1]), epoch_wall_s=wall,
                                         minibatch_counts=[reports[i][0] for i in sorted(reports)],
                                         staleness_mean=mean, staleness_max=mx,
                                         bytes_exchanged=sum(group.bytes_sent),
                                         frames_per_s=frames / wall if wall > 0 else None))
            group.reset_counters()
            for i in range(1, learners + 1):
                go[i].put(True)
            t0 = clock.now()

    actors = []
    for i in range(1, learners + 1):
        actors.append(learner(i))
        actors.append(agent(i))
    actors.append(orchestrator)
    clock.run(actors)
    return RunResult(weights=be.weights(L[1]), records=records,
                     trace={"staleness": staleness, "staleness_by_learner": staleness_by_learner, "backend": be})
