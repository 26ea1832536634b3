"""Synthetic workloads of the BASELINE.json configs (SURVEY.md section 8(d) recipe).

The reference's own generator (``generate_workload``) is not
shipped, so the recipe uses only reference-equivalent pieces: the SPEC.md:162
archetype presets, SplitMix64 jitter from ``substream(7, 1)`` drawn in job
order, two memory tiers and ``build_profile_table`` with the synthetic
executor.  Identical to what ``tests/golden/make_golden.py`` builds from the
reference package itself (the golden tables pin it).
"""

from __future__ import annotations

from .domain import ClusterSpec, JobSpec, NodeSpec, TechniqueSpec, Workload
from .profiling import SyntheticExecutor, build_profile_table
from .rng import substream

# SPEC.md:162 default archetype parameters, registration order = option order.
TECHNIQUES_4 = (
    TechniqueSpec(name="ddp", archetype="replicated", serial_fraction=0.02, comm_overhead=0.01),
    TechniqueSpec(name="fsdp", archetype="sharded", serial_fraction=0.05, comm_overhead=0.03),
    TechniqueSpec(name="gpipe", archetype="pipelined", serial_fraction=0.15, comm_overhead=0.005),
    TechniqueSpec(name="spill", archetype="offloaded", serial_fraction=0.02, comm_overhead=0.01,
                  offload_multiplier=2.5),
)
TECHNIQUES_6 = TECHNIQUES_4 + (
    TechniqueSpec(name="tp", archetype="sharded", serial_fraction=0.08, comm_overhead=0.02),
    TechniqueSpec(name="zero3", archetype="sharded", serial_fraction=0.04, comm_overhead=0.035),
)

# name -> (jobs, nodes, gpus per node, techniques, search mode)
CONFIGS = {
    1: dict(name="cfg1-paper-8job-1x8-exhaustive", jobs=8, nodes=1, gpus=8, techs=TECHNIQUES_4),
    2: dict(name="cfg2-paper-8job-1x8-introspection", jobs=8, nodes=1, gpus=8, techs=TECHNIQUES_4),
    3: dict(name="cfg3-baselines-16job-1x8", jobs=16, nodes=1, gpus=8, techs=TECHNIQUES_4),
    4: dict(name="cfg4-sweep-32job-4x8", jobs=32, nodes=4, gpus=8, techs=TECHNIQUES_4),
    5: dict(name="cfg5-stress-64job-6tech-1x32", jobs=64, nodes=1, gpus=32, techs=TECHNIQUES_6),
}


def synthetic_workload(n_jobs: int, n_nodes: int, gpus_per_node: int, techniques=TECHNIQUES_4,
                       seed: int = 7, gpu_memory: float = 40.0) -> Workload:
    """Two-tier job mix: odd j large (96 GiB model), even j small (20 GiB)."""
    stream = substream(seed, 1)
    jobs = []
    for j in range(n_jobs):
        jitter = 0.9 + 0.2 * stream.uniform()
        large = j % 2 == 1
        jobs.append(JobSpec(
            id=f"j{j:02d}",
            total_batches=10_000 * (1 + j % 3),
            base_batch_time=(4.0 if large else 1.0) * jitter,
            model_memory=96.0 if large else 20.0,
            activation_memory=8.0 if large else 6.0,
        ))
    nodes = tuple(NodeSpec(id=f"n{i}", gpu_count=gpus_per_node, gpu_memory=gpu_memory)
                  for i in range(n_nodes))
    return Workload(jobs=tuple(jobs), cluster=ClusterSpec(nodes=nodes), techniques=tuple(techniques))


def config_workload(k: int):
    """(workload, profile table, config dict) for BASELINE.json config k (1-based)."""
    c = CONFIGS[k]
    w = synthetic_workload(c["jobs"], c["nodes"], c["gpus"], c["techs"])
    return w, build_profile_table(w, SyntheticExecutor(w.cluster)), c


# ---------------------------------------------------------------- SPEC.md:428-436 mirror presets
# Table 1 grid shape: 2 models x 3 learning rates x 2 batch sizes = 12 jobs on `nodes` x 8
# GPUs; one model tier fits a GPU under replication, the other needs sharding / pipelining /
# offloading; +-10 % seeded jitter on the per-batch time.  Numeric job parameters are
# synthetic (the SPEC's own design decision); epochs fold into total_batches.
PRESETS = {
    #                 (model id, model GiB, activation GiB, base s/batch, batches per epoch x 10 epochs)
    "wikitext_mirror": (("gpt2", 20.0, 6.0, 1.0, 2_000), ("gptj", 96.0, 8.0, 4.0, 2_000)),
    "imagenet_mirror": (("resnet200", 12.0, 10.0, 0.8, 2_500), ("vitg", 72.0, 12.0, 3.0, 2_500)),
}


def generate_workload(preset: str, nodes: int = 1, seed: int = 7, gpus_per_node: int = 8) -> Workload:
    """SPEC.md:428-436 generate_workload: 12 jobs (model x lr x batch size) on nodes x 8 GPUs."""
    from . import errors as E

    if preset not in PRESETS:
        raise E.InvariantViolation("preset", f"unknown preset {preset!r}")
    stream = substream(seed, 2)
    jobs = []
    for model, mem, act, base, batches in PRESETS[preset]:
        for lr in range(3):
            for bs, (scale, bfac) in enumerate(((1.0, 1.0), (1.8, 0.5))):   # batch x2: ~1.8x time, half the batches
                jitter = 0.9 + 0.2 * stream.uniform()
                jobs.append(JobSpec(id=f"{model}-lr{lr}-bs{bs}", total_batches=int(batches * 10 * bfac),
                                    base_batch_time=base * scale * jitter, model_memory=mem,
                                    activation_memory=act * scale))
    cluster = ClusterSpec(nodes=tuple(NodeSpec(id=f"n{i}", gpu_count=gpus_per_node, gpu_memory=40.0)
                                      for i in range(nodes)))
    return Workload(jobs=tuple(jobs), cluster=cluster, techniques=TECHNIQUES_4)


def random_workload(seed: int, n_jobs=None, n_nodes=None, gpus_per_node: int = 4) -> Workload:
    """SPEC.md:481 criterion 3 workloads: 4-8 jobs, 1-2 nodes of 4 GPUs, synthetic profiles."""
    s = substream(seed, 3)
    J = n_jobs or 4 + s.below(5)
    N = n_nodes or 1 + s.below(2)
    jobs = []
    for j in range(J):
        large = s.below(3) == 0
        jobs.append(JobSpec(id=f"j{j:02d}", total_batches=1000 * (1 + s.below(10)),
                            base_batch_time=(3.0 if large else 1.0) * (0.5 + s.uniform()),
                            model_memory=60.0 if large else 10.0 + 20.0 * s.uniform(),
                            activation_memory=4.0 + 4.0 * s.uniform()))
    cluster = ClusterSpec(nodes=tuple(NodeSpec(id=f"n{i}", gpu_count=gpus_per_node, gpu_memory=40.0)
                                      for i in range(N)))
    return Workload(jobs=tuple(jobs), cluster=cluster, techniques=TECHNIQUES_4)
