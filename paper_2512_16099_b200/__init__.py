"""B200-native engine for the hot path of the fragmentation-aware online MIG
scheduler of arXiv 2512.16099 ("migsched").

Public surface, shaped like the reference's C++ API (see model.py for the
file:line map):

* ``run(trace, cfg)``               — migsched::run (sim.hpp:114) on the GPU
* ``Engine.run_batch(batch, cfgs)`` — many independent traces, one warp each
* ``Engine.stage(...)``             — HBM-resident batch for benchmarking
* ``generate(spec)``                — migsched::generate (workload.cpp:98-127)
* decision-level ``schedule`` / ``first_fit_schedule`` / ``dispatch_schedule`` /
  ``try_dequeue`` / ``plan_intra`` / ``plan_inter`` / ``on_departure`` /
  ``apply_move`` live in ``decisions``.

Everything on the hot path executes sm_100a kernels from
``libmigsched_b200.so``; there is no CPU fallback.
"""
from .model import (  # noqa: F401
    COMPUTE_SLICES,
    MEMORY_SLICES,
    PROFILE_NAMES,
    START_INDEXES,
    FeatureFlags,
    Job,
    MigschedError,
    SchedulerConfig,
    SimConfig,
    TraceBatch,
    WorkloadSpec,
    find_profile,
    preset,
    preset_names,
    static_layout_preset,
    static_layout_preset_names,
)
from .results import TraceResult, event_to_dict  # noqa: F401


def __getattr__(name):
    # Lazy: importing the package must not require the CUDA library.
    if name in ("Engine", "run", "generate", "generate_batch", "default_engine", "Staged"):
        from . import engine

        return getattr(engine, name)
    raise AttributeError(name)
