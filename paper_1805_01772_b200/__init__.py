"""B200-native in-graph dynamic control flow (arXiv 1805.01772): while_loop / cond compiled to
Switch/Merge/Enter/Exit/NextIteration, stack-based loop gradients, executed by a persistent
sm_100a driver kernel. The C-ABI is include/cf.h; this package is its Python binding."""
from . import cf  # noqa: F401  (raises ImportError if libcf.so is missing: no CPU fallback)
