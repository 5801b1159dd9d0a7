"""B200-native American-option QMC pricer (reference: arxiv/paper_1205_0106 qmc-pricer).

The hot path -- ``qmc::price_american`` and everything it calls -- runs as
hand-written sm_100a CUDA kernels behind the C ABI in ``include/qmcg.h``
(library ``libqmcg.so``, built in-tree by ``build.py``). ``qmcg`` is the
ctypes binding with the reference's names.
"""
from .qmcg import (  # noqa: F401
    Context, ExecPolicy, Method, OptionKind, OptionSpec, PricingResult, backward_sweep, combine_nodes,
    convergence_curve, load_library, mc_european_price, price_american, sweep_value, tree_node_range,
    validate_simulation,
)

__all__ = ["Context", "ExecPolicy", "Method", "OptionKind", "OptionSpec", "PricingResult", "backward_sweep",
           "combine_nodes", "convergence_curve", "load_library", "mc_european_price", "price_american",
           "sweep_value", "tree_node_range", "validate_simulation"]
