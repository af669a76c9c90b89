"""One small 2D assembly (sanitizer / debugging target): python tools/one2d.py <p> <form> <geometry> [sx sy]"""
import sys

sys.path.insert(0, ".")
import paper_1904_06971_b200 as pkg  # noqa: E402

p, form, geom = int(sys.argv[1]), sys.argv[2], sys.argv[3]
spans = (int(sys.argv[4]), int(sys.argv[5])) if len(sys.argv) > 5 else (7, 6)
disc = pkg.make_discretization(pkg.builtin_domain(geom), p, spans)
A = pkg.assemble(pkg.FormKind(form), disc)
print("ok", A.mat.nnz)
