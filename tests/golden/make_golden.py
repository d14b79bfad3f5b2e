"""Generate the golden fixtures in tests/golden/ by running the reference itself.

The reference's proj/core sources are compiled unmodified by oracle/build_ref.sh
(Eigen replaced by the oracle's Eigen-API shim) into
oracle/_ref/libtopmg_ref.so. This script needs that library (and therefore
/root/reference) and is run in the build container; the fixtures it writes are
small and committed, so tests on the GPU box never touch /root/reference.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as O  # noqa: E402
from paper_2410_06850_b200 import inputs  # noqa: E402

CASES = [
    # name, n, ncc, sd, vf, kmin, passes, radius, kind, fine, coarse
    ("c4_n16_k1e-3_mmg_cellcc", 16, 2, 2, 0.3, 1e-3, 3, 2, "mmg", "cell", "cc"),
    ("c4_n16_k1e-6_mmg_cellcc", 16, 2, 2, 0.3, 1e-6, 3, 2, "mmg", "cell", "cc"),
    ("c4_n16_k1e-3_mmg_default", 16, 2, 2, 0.3, 1e-3, 3, 2, "mmg", None, None),
    ("c4_n16_k1e-3_jacobi", 16, 2, 2, 0.3, 1e-3, 3, 2, "jacobi", None, None),
    ("c8_n32_k1e-6_mmg_cellcc", 32, 2, 2, 0.3, 1e-6, 3, 2, "mmg", "cell", "cc"),
    ("c8_n32_k1e-3_jacobi", 32, 2, 2, 0.3, 1e-3, 3, 2, "jacobi", None, None),
]


def main():
    if not O.ref_available():
        raise SystemExit("oracle/_ref/libtopmg_ref.so missing: run bash oracle/build_ref.sh")
    patches = O.bottom_center_patch()
    for name, n, ncc, sd, vf, kmin, passes, radius, kind, fb, cb in CASES:
        rho = inputs.box_filter_design(n, vf, passes=passes, radius=radius)
        kappa = O.ref_conductivity(rho, kmin, 1.0, 3)
        A, rhs = O.ref_assemble(n, kappa, np.ones(n ** 3), patches)
        res, setup = O.ref_solve(n, ncc, sd, kappa, rhs, patches, kind, fb, cb, rtol=1e-8,
                                 maxit=20000)
        x = np.random.default_rng(7).standard_normal(n ** 3)
        np.savez_compressed(
            os.path.join(HERE, name + ".npz"),
            n=n, ncc=ncc, sd=sd, vf=vf, kmin=kmin, passes=passes, radius=radius,
            kind=kind, fine_blocks=str(fb), coarse_blocks=str(cb), rtol=1e-8,
            rho_sum=rho.sum(), rhs=rhs, x=res.x, iterations=res.iterations,
            converged=res.converged, history=res.residual_history,
            apply_in=x, apply_out=A @ x)
        print(name, res.iterations, res.converged)
    # local spectral basis of one coarse cell (coarse_space.cpp:279-304)
    n, ncc, sd = 16, 2, 2
    rho = inputs.box_filter_design(n, 0.3)
    kappa = O.ref_conductivity(rho, 1e-3, 1.0, 3)
    vals, vecs = O.ref_local_basis(n, ncc, sd, kappa, 5, 4)
    np.savez_compressed(os.path.join(HERE, "local_basis_n16_cell5.npz"), n=n, ncc=ncc, sd=sd,
                        kmin=1e-3, cid=5, values=vals, vectors=vecs)
    print("local basis", vals)


if __name__ == "__main__":
    main()
