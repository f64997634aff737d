"""Alias of ``overlap_sim.heuristic``'s module path (drop-in import path); see ``selector.py``."""
from .selector import *  # noqa: F401,F403
from .selector import __dict__ as _src

globals().update({k: v for k, v in _src.items() if not k.startswith("__")})
