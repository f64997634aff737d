"""Alias of ``overlap_sim.engine``'s module path (drop-in import path); see ``simulator.py``."""
from .simulator import *  # noqa: F401,F403
from .simulator import __dict__ as _src

globals().update({k: v for k, v in _src.items() if not k.startswith("__")})
