"""B200-native DPT eigensolver (arXiv:2002.12872): the reference `dynspec` C++
solver API over hand-written sm_100a CUDA kernels (libdpt_b200.so)."""
from .dpt import (ConvergenceReport, ConvergenceStatus, Context, CsrMatrix, DegenerateSpectrum,
                  DeviceError, DominantEigenpair, EigenIterate, IterationOptions, NoDeviceError,
                  PartitionedProblem, Plan, ShapeError, fp64_peak_tflops, SingleRowReport, TraceAborted, check_degenerate,
                  default_context, dominant_eigenpair, effective_window, eigenvalue_of, iterate_fixed,
                  iterate_full, iterate_ramped, iterate_single, spectral_spread, step_full, step_single,
                  to_string, CellClass, ScanGrid, ScanMode, DomainGrid, grid_coordinate, scan_domain, IoError, read_matrix_market, write_matrix_market, homotopy_solve,
                  matmul_dense, solve_linear_multi)

__all__ = [n for n in dir() if not n.startswith("_")]
