"""Alias of ``overlap_sim.planner``'s module path (drop-in import path); see ``routing.py``."""
from .routing import *  # noqa: F401,F403
from .routing import __dict__ as _src

globals().update({k: v for k, v in _src.items() if not k.startswith("__")})
