"""Seeded synthetic fields shaped like the paper's workloads.

This package holds NONE of the estimator's arithmetic: it only draws random
numbers and shapes them into float32 arrays.  It is the one module both the
oracle side (tests) and the CUDA side (tests, bench) import.
"""
from .fields import (CONFIGS, c1_field, c2_field, c3_field, c4_field, c5_field, grf,  # noqa: F401
                     make_field, config_fields)
