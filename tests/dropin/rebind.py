"""The INTEGRATION.md rebinding, verbatim, as a function (test infrastructure): a maintainer of the
reference (`surriga`) installs the B200 path by rebinding the by-name imports of its modules
(surrogate.py:23-33, studies.py:21-50, cli.py:26-41, __init__.py:33-67)."""


def install(only_assemble_in_surrogate=False):
    import surriga
    import surriga.assembly
    import surriga.cli
    import surriga.solvers
    import surriga.studies
    import surriga.surrogate

    import paper_1904_06971_b200 as b200

    def _assemble(form, disc, rows=None, coefficient=1.0):
        A = b200.assemble(form, disc, rows=rows, coefficient=coefficient)
        return surriga.assembly.SparseMatrix(mat=A.mat, symmetric=A.symmetric, populated_rows=A.populated_rows)

    if only_assemble_in_surrogate:
        # the reference's own build_surrogate_matrix, whose quadrature-row call (surrogate.py:588)
        # now runs on the GPU
        surriga.surrogate.assemble = _assemble
        return

    def _surrogate(form, disc, strategy=None, q=3, mode=None, coefficient=1.0):
        A, rep = b200.build_surrogate_matrix(form, disc, strategy, q, mode, coefficient)
        r = surriga.surrogate.AssemblyReport(**{k: getattr(rep, k) for k in rep.__dataclass_fields__})
        return surriga.assembly.SparseMatrix(mat=A.mat, symmetric=A.symmetric), r

    def _divergence(stokes, rows=None):
        D = b200.assemble_divergence(stokes, rows=rows)
        return [surriga.assembly.SparseMatrix(mat=d.mat, symmetric=False, populated_rows=d.populated_rows) for d in D]

    def _surrogate_divergence(stokes, strategy=None, q=3, mode=None):
        D, rep = b200.build_surrogate_divergence(stokes, strategy, q, mode)
        r = surriga.surrogate.AssemblyReport(**{k: getattr(rep, k) for k in rep.__dataclass_fields__})
        return [surriga.assembly.SparseMatrix(mat=d.mat, symmetric=False) for d in D], r

    for mod in (surriga, surriga.assembly, surriga.surrogate, surriga.studies, surriga.cli):
        if hasattr(mod, "assemble"):
            mod.assemble = _assemble
        if hasattr(mod, "build_surrogate_matrix"):
            mod.build_surrogate_matrix = _surrogate
        if hasattr(mod, "assemble_divergence"):
            mod.assemble_divergence = _divergence
        if hasattr(mod, "build_surrogate_divergence"):
            mod.build_surrogate_divergence = _surrogate_divergence
        if hasattr(mod, "assemble_load"):
            mod.assemble_load = b200.assemble_load
        if hasattr(mod, "quadrature_fields"):
            mod.quadrature_fields = b200.quadrature_fields
        if hasattr(mod, "save_matrix_market"):
            mod.save_matrix_market = b200.save_matrix_market

    _ref_solve = surriga.solvers.solve_spd

    def _solve_spd(A, b, opts=None):
        opts = opts or surriga.solvers.SolveOptions()
        if opts.method != "conjugate-gradient":
            return _ref_solve(A, b, opts)
        o = b200.solvers.SolveOptions(opts.method, opts.tolerance, opts.max_iterations, opts.preconditioner)
        return b200.solvers.solve_spd(A, b, o)

    for mod in (surriga, surriga.solvers, surriga.studies, surriga.cli):
        if hasattr(mod, "solve_spd"):
            mod.solve_spd = _solve_spd
