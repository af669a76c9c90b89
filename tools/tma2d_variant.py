"""Run the p=4 polynomial Poisson / p=2 rational bi-Laplacian 2D cases with an experimental build."""
import subprocess
import sys

code = '''
import sys; sys.path.insert(0, sys.argv[4])
import paper_1904_06971_b200 as pkg
p, form, geom = int(sys.argv[1]), sys.argv[2], sys.argv[3]
disc = pkg.make_discretization(pkg.builtin_domain(geom), p, (23, 19))
A = pkg.assemble(pkg.FormKind(form), disc)
print("ok", A.mat.nnz, pkg.__file__)
'''
for root in sys.argv[1:]:
    for p, form, geom in ((4, "poisson", "coons_quadratic"), (3, "poisson", "coons_quadratic"), (3, "poisson", "coons_rational"),
                          (2, "poisson", "coons_quadratic"), (1, "poisson", "coons_quadratic")):
        r = subprocess.run([sys.executable, "-c", code, str(p), form, geom, root], capture_output=True, text=True, timeout=120)
        msg = (r.stdout.strip().splitlines() or [""])[-1] if r.returncode == 0 else (r.stderr.strip().splitlines() or [""])[-1][-100:]
        print(root, p, form, geom, r.returncode, msg, flush=True)
