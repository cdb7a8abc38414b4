"""B200-native exact treewidth (arXiv 1709.09990): the reference elimtw C API
with the Held-Karp wavefront on sm_100a kernels. See DESIGN.md."""
from . import elimtw, generators  # noqa: F401
from .elimtw import (ElimtwError, Graph, Options, ParseError, Result, decide, device_info,  # noqa: F401
                     expand_layer, solve, solve_layers, version)
