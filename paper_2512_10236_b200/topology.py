"""Alias of ``overlap_sim.topology``'s module path (drop-in import path); see ``pricing.py``."""
from .pricing import *  # noqa: F401,F403
from .pricing import __dict__ as _src

globals().update({k: v for k, v in _src.items() if not k.startswith("__")})
