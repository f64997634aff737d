"""Alias of ``overlap_sim.core``'s module path (drop-in import path); see ``domain.py``."""
from .domain import *  # noqa: F401,F403
from .domain import __dict__ as _src

globals().update({k: v for k, v in _src.items() if not k.startswith("__")})
