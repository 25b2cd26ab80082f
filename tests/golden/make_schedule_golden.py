"""Golden schedule vectors produced by the REFERENCE package (run here, where
/root/reference is importable) and committed for the GPU box:

  epoch_minibatches / static_partition index streams, learning-rate values,
  Topology partners, chunk plans, and ADPSGD / SSGD / Hybrid schedules
  (minibatch counts, staleness samples per learner, exchange pairs, virtual
  epoch wall times) under jittered delays with a straggler.

    python tests/golden/make_schedule_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.append("/root/reference/pkg/src")
sys.dont_write_bytecode = True


def main():
    import distsgd as R

    out = {}
    # a1 / a2: index streams
    mb = {}
    for n, B, seed, ep in [(900, 160, 0, 1), (900, 160, 0, 2), (14746, 256, 0, 1), (58982, 160, 7, 3)]:
        data = R.Dataset(inputs=np.zeros((n, 1)), targets=np.zeros(n), train_indices=np.arange(n),
                         heldout_indices=np.arange(0))
        batches = R.epoch_minibatches(data, B, seed, ep)
        mb[f"{n}_{B}_{seed}_{ep}"] = [b.tolist() for b in batches]
    out["epoch_minibatches"] = mb
    from distsgd.engines.ssgd import static_partition

    data = R.Dataset(inputs=np.zeros((900, 1)), targets=np.zeros(900), train_indices=np.arange(900),
                     heldout_indices=np.arange(0))
    out["static_partition_900_160_2"] = [[b.tolist() for b in part]
                                         for part in static_partition(R.epoch_minibatches(data, 160, 0, 1), 2)]
    # a5: learning rates
    lrs = []
    for name, spec in [("large", R.large_batch_schedule()), ("base", R.baseline_schedule(0.1))]:
        for ep in range(1, 17):
            for k, n in [(0, 7), (3, 7), (6, 7), (0, 1)]:
                lrs.append([name, ep, k, n, R.learning_rate(spec, ep, k, n)])
    out["learning_rate"] = lrs
    # a4: partners
    out["partners"] = {str(lam): {str(i): [R.Topology(lam).partner(i, it) for it in range(1, 11)]
                                  for i in R.Topology(lam).senders()} for lam in (2, 4, 8)}
    # a10: chunk plans
    out["chunk_plans"] = {f"{d}_{w}_{c}": list(map(list, R.make_chunk_plan(d, w, c).bounds))
                          for d, w, c in [(10, 3, None), (43130368, 8, None), (7, 4, 6), (100003, 8, 16)]}
    # a13 / a12 / C10: schedules under jittered delays, value-independent
    obj = R.make_objective("quadratic", 2)
    ds = R.make_dataset("quadratic", 600, 2, 1)
    delays = dict(base_compute_s=2e-3, compute_jitter_s=1e-3, comm_latency_s=2e-4, comm_jitter_s=1e-4,
                  slowdowns={3: 2.0}, jitter_seed=5)
    scheds = {}
    for lam in (2, 4, 8):
        res = R.run_adpsgd(obj, ds, R.baseline_schedule(0.05, total_epochs=4), learners=lam, epochs=2,
                           batch_size=16, seed=3, delays=R.DelayModel(**delays), clock=R.VirtualClock(),
                           record_trace=True)
        scheds[f"adpsgd_{lam}"] = {
            "counts": [r.minibatch_counts for r in res.records],
            "wall": [r.epoch_wall_s for r in res.records],
            "exchanges_bytes": [r.bytes_exchanged // (8 * obj.param_dim) for r in res.records],
            "staleness_by_learner": {str(k): v for k, v in res.trace["staleness_by_learner"].items()},
            "pairs": [[e.sender, e.receiver] for e in res.trace["exchanges"]],
        }
    for lam in (2, 4):
        res = R.run_ssgd(obj, ds, R.baseline_schedule(0.05, total_epochs=4), learners=lam, epochs=2, batch_size=16,
                         seed=3, delays=R.DelayModel(**delays), clock=R.VirtualClock())
        scheds[f"ssgd_{lam}"] = {"counts": [r.minibatch_counts for r in res.records],
                                 "wall": [r.epoch_wall_s for r in res.records],
                                 "bytes_per_elem": [r.bytes_exchanged // 8 for r in res.records]}
        res = R.run_hybrid(obj, ds, R.baseline_schedule(0.05, total_epochs=4), learners=lam, epochs=2,
                           batch_size=16, seed=3, delays=R.DelayModel(**delays), clock=R.VirtualClock())
        scheds[f"hybrid_{lam}"] = {"counts": [r.minibatch_counts for r in res.records],
                                   "wall": [r.epoch_wall_s for r in res.records],
                                   "staleness": res.trace["staleness"].samples}
    out["schedules"] = scheds
    out["schedule_delays"] = delays
    with open(os.path.join(HERE, "schedule_golden.json"), "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main()
