"""B200-native (sm_100a) MetaTune cost-model hot path, drop-in for the
reference package `kerntune`'s model / meta / graph-encoding API.

Host logic (knob spaces, graph construction, layouts) is plain Python/numpy;
every batched numeric entry point runs in libkerntune_b200.so (hand-written
CUDA for sm_100a, C-ABI in include/kerntune_b200.h) and raises if the library
is missing.
"""

from .errors import ConfigError, DomainError, NumericError
from .kernels import (
    OP_TYPES,
    KernelSpec,
    KnobConfig,
    KnobDef,
    KnobSpace,
    build_knob_space,
    config_index,
    index_config,
    sample_configs,
)
from .graphs import (
    FEATURE_DIM,
    BatchLayout,
    CodeGraph,
    GraphNode,
    SuperGraphTemplate,
    augment_to_super,
    batch_layout,
    build_super_template,
    config_graph,
    graph_from_text,
    graph_to_tensors,
    graph_to_text,
)
from .util import rng_from, stable_digest

__version__ = "0.1.0"


_LAZY = ("model", "meta", "search", "dist", "dataset")


def __getattr__(name):
    # torch-backed modules load on first use so host-only tooling stays light
    import importlib

    if name.startswith("_") or name in _LAZY:
        raise AttributeError(name)
    for mod in _LAZY:
        try:
            m = importlib.import_module(f".{mod}", __name__)
        except ModuleNotFoundError:
            continue
        if hasattr(m, name):
            return getattr(m, name)
    raise AttributeError(name)
