"""B200-native (sm_100a) drop-in for the hot path of arXiv 1904.06971 (``surriga``):
full-quadrature and surrogate Galerkin assembly of IGA stiffness / mass / bi-Laplacian
matrices into CSR.

Public entry points keep the reference signatures:
    assemble(form, disc, rows=None, coefficient=1.0) -> SparseMatrix
    build_surrogate_matrix(form, disc, strategy=None, q=3, mode=None, coefficient=1.0)
        -> (SparseMatrix, AssemblyReport)
"""
from .assembly import (  # noqa: F401
    Discretization,
    FormKind,
    SparseMatrix,
    StokesSpaces,
    assemble,
    assemble_divergence,
    assemble_divergence_device,
    assemble_load,
    assemble_device,
    elements_for_rows,
    form_is_symmetric,
    gauss_rule,
    is_bitwise_symmetric,
    make_discretization,
    matrices_bitwise_equal,
    quadrature_fields,
    save_matrix_market,
    load_matrix_market,
    set_device,
    stokes_subgrid_spaces,
)
from .geometry import (  # noqa: F401
    BUILTIN_NAMES,
    GeometryMap,
    builtin_domain,
    load_geometry,
    quarter_annulus,
    save_geometry,
    sin_map_standin,
    trivariate_polynomial_3d,
    twisted_cube_standin,
    unit_cube,
    unit_square,
    weights_for_space,
)
from .spaces import NurbsWeights, TensorSpace, make_open_uniform_knots, make_tensor_space  # noqa: F401

try:  # surrogate host layer (added with its kernels)
    from .surrogate import (  # noqa: F401
        AssemblyReport,
        ConstantSampling,
        MeshDependentSampling,
        SurrogateMode,
        build_surrogate_divergence,
        build_surrogate_matrix,
        surrogate_plan,
    )
except ImportError:  # pragma: no cover
    pass

__version__ = "0.1.0"
