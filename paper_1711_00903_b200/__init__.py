"""B200-native BP1.0 / BP3.5 / BP3.0 hexahedral element matvecs (arXiv 1711.00903).

Drop-in for the operator path of the reference ``hexbench`` package: the same
public names (``make_operator``, ``apply_operator``, ``FieldVector``, ...)
backed by hand-written sm_100a kernels behind the C ABI in
``include/hexbench_b200.h``.
"""

from .basis import (MAX_DEGREE, OperatorMatrix, contract_dim, diff_matrix_gl, diff_matrix_gll,
                    interp_matrix)
from .mesh import (FACTOR_NAMES, DegenerateGeometryError, GeometricFactors, HexMesh,
                   build_cube_mesh, geometric_factors, perturb_mesh, trilinear_jacobian,
                   trilinear_map)
from .operators import (AccessCounters, FieldVector, OperatorInstance, UnsupportedVariantError,
                        apply_baseline, apply_bp1, apply_bp3, apply_bp35, apply_device, apply_host,
                        apply_operator, interpolate_to_gl, make_operator,
                        project_to_gll)
from .perf import (BENCHMARKS, BP1, BP3, BP35, VARIANTS, BandwidthCalibration, RooflinePoint,
                   RooflineSeries, measure_stream_bandwidth,
                   TrafficModel, element_counters, flop_model, roofline_global,
                   roofline_series, roofline_shared, scratch_traffic, shared_bandwidth_ansatz,
                   traffic)
from .quadrature import (QuadratureRule, check_rule, gl_rule, gll_rule, lagrange_deriv,
                         lagrange_eval, legendre_and_derivative)

__version__ = "0.1.0"
