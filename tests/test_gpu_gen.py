"""Seeded synthetic designs generated on the device (gen.cu) are bit-identical
to inputs.box_filter_design (itself bit-identical to the oracle's C
generator), including the top-k tie rule (rng.cpp:39-51)."""
import numpy as np
import pytest

import oracle as O
from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, inputs

pytestmark = pytest.mark.gpu
BC = BoundarySpec.bottom_center_patch(1.0, 1.0, 0.2, 0.0)


@pytest.mark.parametrize("dims,ncc,sd,vf,passes,radius,seed", [
    ((16, 16, 16), 2, 2, 0.3, 3, 2, 20240501),
    ((16, 24, 32), (2, 3, 4), 2, 0.25, 2, 1, 7),
    ((64, 64, 64), 4, 2, 0.3, 3, 2, 20240501),   # BASELINE configs[0]
    ((32, 32, 32), 2, 2, 0.2, 3, 4, 20240501),   # configs[3] generator at 32^3
    ((16, 16, 16), 2, 2, 0.3, 0, 2, 99),         # raw uniforms
    ((8, 8, 8), 1, 2, 0.37, 1, 8, 3),            # window = whole domain: all values tie
    ((8, 16, 16), (1, 2, 2), 2, 0.41, 1, 4, 5),  # x-window covers x: ties in rows of 8
])
def test_generated_design_bitwise(dims, ncc, sd, vf, passes, radius, seed):
    nx, ny, nz = dims
    ref = inputs.box_filter_design(dims, vf, seed=seed, passes=passes, radius=radius)
    c = Context(GridSpec(nx, ny, nz), ncc, sd)
    rho = c.set_design_generated(vf, 1e-3, boundary=BC, seed=seed, passes=passes, radius=radius,
                                 return_rho=True)
    np.testing.assert_array_equal(rho, ref)
    assert rho.sum() == min(nx * ny * nz, int(np.ceil(vf * nx * ny * nz)))
    # the context now holds kappa(rho): same operator as set_design(rho)
    x = np.random.default_rng(1).standard_normal(nx * ny * nz)
    c2 = Context(GridSpec(nx, ny, nz), ncc, sd)
    c2.set_design(ref, 1e-3, 1.0, 3, BC)
    np.testing.assert_array_equal(c.apply_operator(x), c2.apply_operator(x))


def test_generated_config0_solid_count():
    c = Context(GridSpec(64, 64, 64), 4, 2)
    rho = c.set_design_generated(0.3, 1e-3, boundary=BC, return_rho=True)
    assert int(rho.sum()) == 78644
    np.testing.assert_array_equal(rho, O.box_filter_design(O.grid(64), 0.3))
