"""thermiga-b200: B200-native hot path of the semi-analytical IGA thermal solver.

The product is ``_lib/libthermiga_b200.so`` (sm_100a CUDA kernels + host C++
behind the C ABI ``include/thermiga_b200.h``); this package is its Python
binding and the seeded BASELINE workloads.
"""
from .api import (ConfigError, Context, CudaError, LaserSpec, Material, NumericError, ScanPath,
                  Simulation,
                  SuperposeOptions, ThermigaError, discretize_scan, elevate_geometry,
                  export_profile_csv,
                  integrated_abs_flux, lib, superpose)

__all__ = ["ConfigError", "Context", "CudaError", "LaserSpec", "Material", "NumericError",
           "ScanPath", "Simulation", "SuperposeOptions", "ThermigaError", "discretize_scan",
           "elevate_geometry",
           "export_profile_csv", "integrated_abs_flux", "lib", "superpose"]
