"""Load callables used by the load-vector goldens and tests (f(x) with x of shape (..., n))."""
import numpy as np

LOAD_FUNCS = {
    "one": lambda x: np.ones(x.shape[:-1]),
    "poly_sin": lambda x: 1.0 + x[..., 0] ** 2 + np.sin(x[..., 1]),
    "prod_cos": lambda x: x[..., 0] * x[..., 1] + np.cos(x[..., 2]),
}
