"""``lpic`` -- the reference package's import name, served by the B200 build.

Code and tests written against /root/reference/pkg/src/lpic (``import lpic``,
``from lpic.codec import encode``, ``from lpic import kernels``) resolve to
paper_2212_01185_b200: every ``lpic.<module>`` below is the corresponding
module of this package (registered in sys.modules, so submodule imports
work), and the top-level names are the package's public API
(reference __init__.py:11-26).
"""

import importlib as _importlib
import sys as _sys

import paper_2212_01185_b200 as _impl
from paper_2212_01185_b200 import *  # noqa: F401,F403

_MODULES = ("codec", "coder", "errors", "kernels", "mixture", "network", "schedules", "synthetic", "training",
            "images", "cli", "verification", "tiles", "shard", "synth")
for _name in _MODULES:
    _mod = _importlib.import_module(f"paper_2212_01185_b200.{_name}")
    _sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod

__version__ = _impl.__version__
__all__ = [n for n in dir(_impl) if not n.startswith("_")]
