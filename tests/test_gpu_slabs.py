"""Partitioned (multi-slab) data path on one GPU.

tmg_create_slabs splits the grid into z-slabs of whole cc-element layers with
ghost brick layers, halo exchanges, cross-slab CG reductions, and a row-block
A_cc^-1 GEMV per slab: everything the NCCL (one slab per GPU) path runs except
the transport. The smoother blocks never straddle slabs, so the partitioned
solve is the same algorithm as the single-slab one: the operator must agree
bit for bit, the preconditioner and the PCG result up to summation order.
"""
import numpy as np
import pytest

from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, inputs

pytestmark = pytest.mark.gpu

PATCH = BoundarySpec.bottom_center_patch(1, 1, 0.2, 0)


def _ctx(n, ncc, sd, kappa, slabs, kind="mmg"):
    from paper_2410_06850_b200 import MmgOptions
    c = Context(GridSpec(n, n, n), ncc, sd, slabs=slabs)
    c.set_conductivity(kappa, PATCH)
    c.setup(kind, MmgOptions(fine_blocks="coarse_cell"))
    return c


def _problem(n, kmin, seed=7):
    """BASELINE-style design (seeded box-filtered field, volume fraction 0.3)."""
    return inputs.conductivity(inputs.box_filter_design(n, 0.3, seed=seed), kmin)


@pytest.mark.parametrize("n,ncc,sd,slabs", [(32, 4, 2, 2), (32, 4, 2, 4), (64, 4, 2, 2),
                                            (64, 4, 2, 4), (64, 8, 1, 8)])
def test_slab_operator_bitwise(n, ncc, sd, slabs):
    kappa = _problem(n, 1e-3)
    a = Context(GridSpec(n, n, n), ncc, sd)
    a.set_conductivity(kappa, PATCH)
    b = Context(GridSpec(n, n, n), ncc, sd, slabs=slabs)
    b.set_conductivity(kappa, PATCH)
    x = np.random.default_rng(1).standard_normal(n ** 3)
    np.testing.assert_array_equal(a.apply_operator(x), b.apply_operator(x))
    np.testing.assert_array_equal(a.assemble_rhs(np.ones(n ** 3)), b.assemble_rhs(np.ones(n ** 3)))


@pytest.mark.parametrize("n,ncc,sd,slabs,kmin", [(32, 4, 2, 2, 1e-3), (32, 4, 2, 4, 1e-6),
                                                 (64, 4, 2, 4, 1e-3), (128, 8, 2, 8, 1e-6)])
def test_slab_preconditioner_matches_single(n, ncc, sd, slabs, kmin):
    kappa = _problem(n, kmin)
    a = _ctx(n, ncc, sd, kappa, 1)
    b = _ctx(n, ncc, sd, kappa, slabs)
    r = np.random.default_rng(3).standard_normal(n ** 3)
    za, zb = a.apply_preconditioner(r), b.apply_preconditioner(r)
    # same blocks and bases; only the A_cc^-1 GEMV sums in another order
    assert np.linalg.norm(za - zb) <= 1e-9 * np.linalg.norm(za)


@pytest.mark.parametrize("n,ncc,sd,slabs,kmin", [(32, 4, 2, 2, 1e-3), (64, 4, 2, 4, 1e-6),
                                                 (128, 8, 2, 8, 1e-6)])
def test_slab_pcg_matches_single(n, ncc, sd, slabs, kmin):
    kappa = _problem(n, kmin)
    a = _ctx(n, ncc, sd, kappa, 1)
    b = _ctx(n, ncc, sd, kappa, slabs)
    rhs = a.assemble_rhs(np.ones(n ** 3))
    ra, rb = a.pcg(rhs, rtol=1e-8), b.pcg(rhs, rtol=1e-8)
    assert ra.report.converged and rb.report.converged
    assert abs(ra.report.iterations - rb.report.iterations) <= 1
    assert np.linalg.norm(ra.x - rb.x) <= 1e-8 * np.linalg.norm(ra.x)


def test_slab_pcg_configs0_matches_single_and_warm_start():
    n = 64
    rho = inputs.box_filter_design(n, 0.3)
    kappa = inputs.conductivity(rho, 1e-3)
    a = _ctx(n, 4, 2, kappa, 1)
    b = _ctx(n, 4, 2, kappa, 4)
    rhs = a.assemble_rhs(np.ones(n ** 3))
    ra, rb = a.pcg(rhs, rtol=1e-8), b.pcg(rhs, rtol=1e-8)
    assert ra.report.iterations == rb.report.iterations
    assert np.linalg.norm(ra.x - rb.x) <= 1e-9 * np.linalg.norm(ra.x)
    # warm start from a perturbed solution: fewer iterations, same answer
    x0 = ra.x * (1 + 1e-3 * np.random.default_rng(5).standard_normal(n ** 3))
    wa, wb = a.pcg(rhs, rtol=1e-8, x0=x0), b.pcg(rhs, rtol=1e-8, x0=x0)
    assert wa.report.iterations == wb.report.iterations < ra.report.iterations
    assert np.linalg.norm(wa.x - wb.x) <= 1e-9 * np.linalg.norm(wa.x)


@pytest.mark.parametrize("kind", ["jacobi", "none"])
def test_slab_baseline_preconditioners(kind):
    n = 32
    kappa = _problem(n, 1e-2)
    a = _ctx(n, 4, 2, kappa, 1, kind)
    b = _ctx(n, 4, 2, kappa, 4, kind)
    rhs = a.assemble_rhs(np.ones(n ** 3))
    ra, rb = a.pcg(rhs, rtol=1e-6, max_iterations=5000), b.pcg(rhs, rtol=1e-6, max_iterations=5000)
    # hundreds of CG steps: summation-order drift moves the count by < 2 %
    assert abs(ra.report.iterations - rb.report.iterations) <= max(1, 0.02 * ra.report.iterations)
    assert np.linalg.norm(ra.x - rb.x) <= 1e-6 * np.linalg.norm(ra.x)


def test_slab_count_must_divide_cc_layers():
    from paper_2410_06850_b200 import ConfigError
    with pytest.raises(ConfigError):
        Context(GridSpec(32, 32, 32), 4, 2, slabs=3)


@pytest.mark.parametrize("kind,fine,planes", [("mmg", "coarse_cell", "0"), ("mmg", "cc", "0"),
                                              ("block_jacobi", "coarse_cell", "0"),
                                              ("two_grid", "coarse_cell", "0"),
                                              ("mmg", "coarse_cell", "1")])
def test_nccl_transport_single_rank(kind, fine, planes):
    """The NCCL transport on a one-rank communicator (TMG_FORCE_DIST=1): the
    partitioned path with all-reduce / all-gather and NCCL calls captured in
    the iteration graph must reproduce the single-GPU solve. planes = 1: A_cc
    as the block Thomas over cc-element z-planes (all-gathered plane blocks,
    replicated plane solve)."""
    import json
    import os
    import subprocess
    import sys
    code = (
        "import json, numpy as np\n"
        "from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, MmgOptions, inputs\n"
        "n = 64\n"
        "k = inputs.conductivity(inputs.box_filter_design(n, 0.3), 1e-3)\n"
        "c = Context(GridSpec(n, n, n), 4, 2)\n"
        "c.set_conductivity(k, BoundarySpec.bottom_center_patch(1, 1, 0.2, 0))\n"
        f"c.setup('{kind}', MmgOptions(fine_blocks='{fine}'))\n"
        "b = c.assemble_rhs(np.ones(n ** 3))\n"
        "r = c.pcg(b, rtol=1e-8, max_iterations=5000)\n"
        "z = c.apply_preconditioner(b)\n"
        "print(json.dumps([r.report.iterations, r.x[::997].tolist(), z[::991].tolist()]))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for force in ("0", "1"):
        env = dict(os.environ, TMG_FORCE_DIST=force, TMG_ACC_PLANES=planes, PYTHONPATH=root)
        p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        out[force] = json.loads(p.stdout.strip().splitlines()[-1])
    assert out["0"][0] == out["1"][0]
    np.testing.assert_allclose(out["1"][1], out["0"][1], rtol=1e-9)
    np.testing.assert_allclose(out["1"][2], out["0"][2], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("kind,fine", [("block_jacobi", None), ("two_grid", "coarse_cell"),
                                       ("mmg", "cc"), ("two_grid", "cc")])
@pytest.mark.parametrize("n,ncc,sd,slabs", [(32, 2, 2, 2), (64, 4, 2, 4)])
def test_slab_variants_match_single(kind, fine, n, ncc, sd, slabs):
    """block_jacobi, two_grid and the reference's cc-element fine blocks on
    slabs (the blocks are whole cc elements, never straddling a slab)."""
    from paper_2410_06850_b200 import MmgOptions
    kappa = _problem(n, 1e-3)
    opts = MmgOptions(fine_blocks=fine) if fine else MmgOptions()
    ctxs = []
    for s in (1, slabs):
        c = Context(GridSpec(n, n, n), ncc, sd, slabs=s)
        c.set_conductivity(kappa, PATCH)
        c.setup(kind, opts)
        ctxs.append(c)
    a, b = ctxs
    r = np.random.default_rng(5).standard_normal(n ** 3)
    za, zb = a.apply_preconditioner(r), b.apply_preconditioner(r)
    assert np.linalg.norm(za - zb) <= 1e-9 * np.linalg.norm(za)
    rhs = a.assemble_rhs(np.ones(n ** 3))
    ra, rb = a.pcg(rhs, rtol=1e-8, max_iterations=5000), b.pcg(rhs, rtol=1e-8, max_iterations=5000)
    assert ra.report.converged and rb.report.converged
    assert abs(ra.report.iterations - rb.report.iterations) <= max(1, ra.report.iterations // 50)
    assert np.linalg.norm(ra.x - rb.x) <= 1e-7 * np.linalg.norm(ra.x)


@pytest.mark.parametrize("n,ncc,sd,slabs,kmin", [(32, 4, 2, 2, 1e-3), (64, 4, 2, 4, 1e-6),
                                                 (64, 4, 2, 2, 1e-3)])
def test_slab_acc_planes_match_single(n, ncc, sd, slabs, kmin, monkeypatch):
    """A_cc as the block Thomas over cc-element z-planes on partitioned
    contexts (each slab assembles its planes, the factors cover every plane,
    the plane solve runs once on the gathered r_cc) against the single-slab
    plane solve (same factors: summation order only) and the dense A_cc^-1
    (another direct solver: PCG parity)."""
    kappa = _problem(n, kmin)
    dense = _ctx(n, ncc, sd, kappa, 1)
    monkeypatch.setenv("TMG_ACC_PLANES", "1")
    single = _ctx(n, ncc, sd, kappa, 1)
    part = _ctx(n, ncc, sd, kappa, slabs)
    r = np.random.default_rng(9).standard_normal(n ** 3)
    zs, zp = single.apply_preconditioner(r), part.apply_preconditioner(r)
    assert np.linalg.norm(zs - zp) <= 1e-9 * np.linalg.norm(zs)
    rhs = dense.assemble_rhs(np.ones(n ** 3))
    rd, rp = dense.pcg(rhs, rtol=1e-8), part.pcg(rhs, rtol=1e-8)
    assert rd.report.converged and rp.report.converged
    assert abs(rd.report.iterations - rp.report.iterations) <= 1
    assert np.linalg.norm(rd.x - rp.x) <= 1e-7 * np.linalg.norm(rd.x)


@pytest.mark.parametrize("slabs", [2, 4])
def test_row_distributed_acc_planes(monkeypatch, slabs):
    """A_cc's plane block Thomas with each slab keeping only its row block of
    every plane inverse (TMG_ACC_ROWS=1, the default from 4 ranks; an
    all-gather of each plane's rows per step under NCCL): the same
    preconditioner and PCG as the replicated plane solve on one slab."""
    from paper_2410_06850_b200 import MmgOptions
    n, ncc, sd = 64, 4, 2
    kappa = _problem(n, 1e-6)
    monkeypatch.setenv("TMG_ACC_PLANES", "1")
    out = []
    for s, rows in ((1, "0"), (slabs, "1")):
        monkeypatch.setenv("TMG_ACC_ROWS", rows)
        c = Context(GridSpec(n, n, n), ncc, sd, slabs=s)
        c.set_conductivity(kappa, PATCH)
        c.setup("mmg", MmgOptions(fine_blocks="coarse_cell"))
        r = np.random.default_rng(8).standard_normal(n ** 3)
        b = c.assemble_rhs(np.ones(n ** 3))
        out.append((c.apply_preconditioner(r), c.pcg(b, rtol=1e-8, max_iterations=3000)))
    (za, ra), (zb, rb) = out
    assert np.linalg.norm(za - zb) <= 1e-9 * np.linalg.norm(za)
    assert abs(ra.report.iterations - rb.report.iterations) <= 1
    assert np.linalg.norm(ra.x - rb.x) <= 1e-7 * np.linalg.norm(ra.x)
