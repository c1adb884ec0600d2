"""pytest plugin: make ``import hetsim`` resolve to this package so the
reference's own unit/acceptance suite can be run against the drop-in
(tests/test_reference_suite.py).  Only used in the build container, where
/root/reference exists; nothing is copied from it."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import paper_1402_6601_b200 as _pkg  # noqa: E402
from paper_1402_6601_b200 import cli, graph, kernels, perfmodel, platform, sched, sim  # noqa: E402,F401

sys.modules["hetsim"] = _pkg
for _name in ("cli", "graph", "kernels", "perfmodel", "platform", "sched", "sim"):
    sys.modules["hetsim." + _name] = getattr(_pkg, _name)
