"""Seeded synthetic instance generator shared by the oracle and the CUDA path's callers.

Holds none of the method's arithmetic (see generate.py's header).
"""
from .generate import Instance, build, gen_config, CONFIGS, selected_inverse, product_on_E, direction_G  # noqa: F401
