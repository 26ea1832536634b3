"""Generate tests/golden/*.json by running the REFERENCE package (jointsched) itself.

Run in the build container, where /root/reference exists:
    python tests/golden/make_golden.py
The GPU box never runs this; tests only read the committed JSON.

What is pinned (all produced by reference code, /root/reference/pkg/src/jointsched):
  * rng vectors: SplitMix64 / below / shuffle / substream / uniform (rng.py:20-56)
  * SPEC.md known answers evaluated by reference code
  * per workload: feasible_configs order (core.py:165-182), build_profile_table entries
    and profiling_cost (profiling.py:122-144), feasible_entries (profiling.py:154-161),
    estimate_runtime at total_batches (profiling.py:147-151)
  * check_plan verdicts on valid and invalid plans (core.py:226-287)
Plus the independent optimum of small instances from HiGHS (scipy.optimize.milp on the
time-indexed MILP of SPEC.md:182-200, built by oracle/saturn_oracle.py) -- not reference
output, recorded separately under "milp".
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from jointsched import core, profiling, rng  # noqa: E402
from jointsched import errors as ref_errors  # noqa: E402

from oracle import saturn_oracle as O  # noqa: E402


def fhex(x: float) -> str:
    return "inf" if math.isinf(x) else float(x).hex()


def techniques(n=4, min_gpus_pipe=1):
    base = [
        core.TechniqueSpec(name="ddp", archetype="replicated", serial_fraction=0.02, comm_overhead=0.01),
        core.TechniqueSpec(name="fsdp", archetype="sharded", serial_fraction=0.05, comm_overhead=0.03),
        core.TechniqueSpec(name="gpipe", archetype="pipelined", serial_fraction=0.15, comm_overhead=0.005,
                           min_gpus=min_gpus_pipe),
        core.TechniqueSpec(name="spill", archetype="offloaded", serial_fraction=0.02, comm_overhead=0.01,
                           offload_multiplier=2.5),
    ]
    if n == 6:
        base += [
            core.TechniqueSpec(name="tp", archetype="sharded", serial_fraction=0.08, comm_overhead=0.02),
            core.TechniqueSpec(name="zero3", archetype="sharded", serial_fraction=0.04, comm_overhead=0.035),
        ]
    return tuple(base)


def recipe(n_jobs, nodes, ntech=4, seed=7, mems=None, min_gpus_pipe=1):
    """SURVEY.md 8(d) recipe, built from reference types and the reference rng."""
    r = rng.substream(seed, 1)
    jobs = []
    for j in range(n_jobs):
        jit = 0.9 + 0.2 * r.uniform()
        big = j % 2 == 1
        jobs.append(core.JobSpec(id=f"j{j:02d}", total_batches=10000 * (1 + j % 3),
                                 base_batch_time=(4.0 if big else 1.0) * jit,
                                 model_memory=96.0 if big else 20.0, activation_memory=8.0 if big else 6.0))
    mems = mems or [40.0] * len(nodes)
    cl = core.ClusterSpec(nodes=tuple(core.NodeSpec(id=f"n{i}", gpu_count=g, gpu_memory=m)
                                      for i, (g, m) in enumerate(zip(nodes, mems))))
    return core.Workload(jobs=tuple(jobs), cluster=cl, techniques=techniques(ntech, min_gpus_pipe))


WORKLOADS = {
    "cfg1": dict(n_jobs=8, nodes=[8]),
    "cfg3": dict(n_jobs=16, nodes=[8]),
    "cfg4": dict(n_jobs=32, nodes=[8, 8, 8, 8]),
    "cfg5": dict(n_jobs=64, nodes=[32], ntech=6),
    "small5_1x4": dict(n_jobs=5, nodes=[4]),
    "small4_2x2": dict(n_jobs=4, nodes=[2, 2]),
    "hetero6": dict(n_jobs=6, nodes=[8, 4], mems=[40.0, 80.0], min_gpus_pipe=2),
    "tiny3_1x3": dict(n_jobs=3, nodes=[3]),
}


def workload_record(w):
    table = profiling.build_profile_table(w, profiling.SyntheticExecutor(w.cluster))
    rec = {
        "workload": json.loads(w.model_dump_json()),
        "entries": [[k[0], k[1], k[2], fhex(v)] for k, v in table.entries.items()],
        "profiling_cost": fhex(table.profiling_cost),
        "feasible_configs": {j.id: [[c.technique, c.gpus] for c in core.feasible_configs(j, w.cluster, w.techniques)]
                             for j in w.jobs},
        "feasible_entries": {j.id: [[c.technique, c.gpus, fhex(lat)] for c, lat in
                                    profiling.feasible_entries(table, j, w)] for j in w.jobs},
        "runtime_total": {j.id: [fhex(profiling.estimate_runtime(table, j, c, j.total_batches))
                                 for c, _ in profiling.feasible_entries(table, j, w)] for j in w.jobs},
    }
    return rec, table


def rng_vectors():
    s = rng.SplitMix64(0)
    v = {"splitmix0_first3": [hex(s.next_u64()) for _ in range(3)]}
    s = rng.SplitMix64(7)
    v["below10_seed7"] = [s.below(10) for _ in range(10)]
    s = rng.SplitMix64(7)
    items = list(range(8))
    s.shuffle(items)
    v["shuffle8_seed7"] = items
    v["substream_7_1_2_first"] = hex(rng.substream(7, 1, 2).next_u64())
    s = rng.substream(7, 1)
    v["uniform_substream_7_1_first64"] = [fhex(s.uniform()) for _ in range(64)]
    # plan_random-style draws on radices (below per job, then shuffle) for a few seeds
    v["random_draws"] = []
    for seed in (0, 1, 7, 12345, 2**63 + 5):
        s = rng.SplitMix64(seed)
        radix = [3, 7, 1, 5, 192, 2]
        opts = [s.below(r) for r in radix]
        order = list(range(len(radix)))
        s.shuffle(order)
        v["random_draws"].append({"seed": str(seed), "radix": radix, "opts": opts, "order": order})
    for salt in (0, 1, 99, 2**40 + 3):
        st = rng.substream(7, salt)
        radix = [4, 7, 5, 6, 5, 8, 4, 6]
        opts = [st.below(r) for r in radix]
        order = list(range(8))
        st.shuffle(order)
        v["random_draws"].append({"substream": [7, salt], "radix": radix, "opts": opts, "order": order})
    return v


def spec_examples():
    out = {}
    job = core.JobSpec(id="a", total_batches=10000, base_batch_time=1.0, model_memory=1.0)
    t = core.TechniqueSpec(name="t", archetype="sharded", serial_fraction=0.2, comm_overhead=0.01)
    out["latency_0.43"] = fhex(profiling.synthetic_latency(job, t, 4, 100.0))
    t3 = core.TechniqueSpec(name="o", archetype="offloaded", serial_fraction=0.0, comm_overhead=0.0,
                            offload_multiplier=3.0)
    out["latency_offload_3"] = fhex(profiling.synthetic_latency(job, t3, 1, 100.0))
    tab = profiling.ProfileTable({("a", "t", 4): profiling.synthetic_latency(job, t, 4, 100.0)}, "synthetic")
    out["estimate_4300"] = fhex(profiling.estimate_runtime(tab, job, core.RunConfig(technique="t", gpus=4), 10000))
    j32 = core.JobSpec(id="m", total_batches=1, base_batch_time=1.0, model_memory=32.0, activation_memory=4.0)
    sh = core.TechniqueSpec(name="s", archetype="sharded", serial_fraction=0.0, comm_overhead=0.0)
    rp = core.TechniqueSpec(name="r", archetype="replicated", serial_fraction=0.0, comm_overhead=0.0)
    of = core.TechniqueSpec(name="o", archetype="offloaded", serial_fraction=0.0, comm_overhead=0.0)
    j500 = core.JobSpec(id="b", total_batches=1, base_batch_time=1.0, model_memory=500.0)
    out["memory"] = [core.memory_feasible(j32, sh, 4, 12.0), core.memory_feasible(j32, rp, 8, 12.0),
                     core.memory_feasible(j500, of, 1, 12.0)]
    return out


def plan_verdicts(w, table):
    """check_plan on hand-made plans: sequential (valid), all-at-0 (capacity), low predicted."""
    out = []
    fe = {j.id: profiling.feasible_entries(table, j, w) for j in w.jobs}
    node = w.cluster.nodes[0]
    for kind in ("sequential", "overlap", "low_predicted", "missing_job"):
        entries, runtimes, t = {}, {}, 0.0
        for job in w.jobs:
            cfg, lat = max(fe[job.id], key=lambda e: (e[0].gpus <= node.gpu_count, e[0].gpus))
            rt = job.total_batches * lat
            start = 0.0 if kind == "overlap" else t
            entries[job.id] = core.PlanEntry(config=cfg, node=node.id, start_time=start)
            runtimes[job.id] = rt
            t += rt
        if kind == "missing_job":
            entries.pop(w.jobs[0].id)
        pred = t * (0.5 if kind == "low_predicted" else 1.0)
        plan = core.Plan(entries=entries, predicted_makespan=pred)
        try:
            core.check_plan(plan, w, runtimes)
            verdict = "ok"
        except ref_errors.SchedulerError as exc:
            verdict = type(exc).__name__
        out.append({"kind": kind,
                    "entries": {k: [e.config.technique, e.config.gpus, e.node, fhex(e.start_time)]
                                for k, e in entries.items()},
                    "predicted": fhex(pred), "runtimes": {k: fhex(v) for k, v in runtimes.items()},
                    "verdict": verdict})
    return out


def milp_small():
    """HiGHS optimum (intervals) of the oracle problems of the small workloads and of config 3
    (whose optimum the local search reaches but the simple lower bound cannot prove)."""
    out = {}
    for name in ("cfg1", "cfg3", "small5_1x4", "small4_2x2", "hetero6", "tiny3_1x3"):
        spec = WORKLOADS[name]
        w = recipe(**spec)
        table = profiling.build_profile_table(w, profiling.SyntheticExecutor(w.cluster))
        prob = O.build(table.entries, w)
        out[name] = {"delta": fhex(prob.delta), "radix": prob.radix, "optimum_intervals": O.milp_optimum(prob)}
    return out


def digest(obj) -> str:
    """sha256 of the canonical JSON of a record section (large workloads are pinned by digest)."""
    return hashlib.sha256(json.dumps(obj, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


BIG = ("cfg3", "cfg4", "cfg5")   # pinned by digests + counts to keep the fixture small


def main():
    gold = {"rng": rng_vectors(), "spec": spec_examples(), "workloads": {}}
    for name, spec in WORKLOADS.items():
        w = recipe(**spec)
        rec, table = workload_record(w)
        if name in ("cfg1", "small4_2x2", "hetero6"):
            rec["check_plan"] = plan_verdicts(w, table)
        if name in BIG:
            rec = {"workload": rec["workload"], "profiling_cost": rec["profiling_cost"],
                   "n_entries": len(rec["entries"]),
                   "n_finite": sum(1 for e in rec["entries"] if e[3] != "inf"),
                   "sha256": {k: digest(rec[k]) for k in
                              ("entries", "feasible_configs", "feasible_entries", "runtime_total")}}
        gold["workloads"][name] = rec
    gold["milp"] = milp_small()
    with open(os.path.join(HERE, "reference_golden.json"), "w") as f:
        json.dump(gold, f, indent=0, sort_keys=True)
    print("wrote", os.path.join(HERE, "reference_golden.json"))


if __name__ == "__main__":
    main()
