"""B200-native (sm_100a) Generalized Neighborhood Attention forward (arXiv 2504.16922).

The product is the C-ABI library ``libgna_b200.so`` (include/gna.h); this
package is its thin ctypes binding.  Build with ``__graft_entry__.build()`` or
``python -m paper_2504_16922_b200.build``.
"""
from .gna import (GnaError, attention_permuted, debug_visits, debug_windows, debug_worklist, device_supported,
                  forward, load, permute, plan_info, release_workspace, unpermute, version, workspace_size)

__all__ = ["GnaError", "attention_permuted", "debug_visits", "debug_windows", "debug_worklist", "device_supported",
           "forward", "load", "permute", "plan_info", "release_workspace", "unpermute", "version",
           "workspace_size"]
