"""Seeded synthetic workloads (test + bench infrastructure).

This package is the ONLY code shared by the oracle side and the CUDA side: it
draws the inputs both receive.  It holds none of the method's arithmetic (no
operator, lumping, Poisson solve or wBFBT step) -- only the paper's benchmark
coefficient (multi-sinker viscosity, Sec. 2.1) sampled at
the points where the library expects it, and U(-1,1) vectors.
"""
from .multisinker import (CONFIGS, Config, sizes, gauss_points_1d, sinker_centers,
                          chi, viscosity, viscosity_at_quadrature, forcing_at_quadrature, make_inputs)

__all__ = ["CONFIGS", "Config", "sizes", "gauss_points_1d", "sinker_centers", "chi",
           "viscosity", "viscosity_at_quadrature", "forcing_at_quadrature", "make_inputs"]
