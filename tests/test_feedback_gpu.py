"""GPU tier: the device-resident feedback loop --
advance T += tend_T, q += tend_q, check_finite and the error-growth envelope
(validate.cpp:113-206) -- against the reference's own error_growth
(oracle/_ref, validate.cpp compiled in place) and against host restatements
of advance / rms_diff on the device's own tendencies."""
import numpy as np
import pytest

import oracle as O
import paper_1711_00289_b200 as P
from paper_1711_00289_b200 import gridgen as G

pytestmark = pytest.mark.gpu


def host_rms(a, b):
    """rms_diff (validate.cpp:41-51) in the reference's AoS order."""
    d = (a - b).T.ravel()
    acc = 0.0
    for x in d:
        acc += x * x
    return np.sqrt(acc / d.size)


@pytest.mark.parametrize("kernel", [P.DEEP, P.SHALLOW])
def test_timestep_equals_convect_plus_host_advance(ctx, kernel):
    s, T, q = G.make_config("c1", n=700, seed=21)
    T1, q1 = T.copy(), q.copy()
    for _ in range(3):   # advance (validate.cpp:127-136) on the host from device tendencies
        deep, sh = ctx.convect(s, T1, q1, kernels=kernel)
        o = deep if kernel == P.DEEP else sh
        T1 = T1 + o.tend_T
        q1 = q1 + o.tend_q
    T2, q2 = ctx.timestep(s, T, q, kernel=kernel, n_steps=3)
    assert np.array_equal(T1, T2) and np.array_equal(q1, q2)
    assert np.array_equal(T, G.make_config("c1", n=700, seed=21)[1])   # input untouched


@pytest.mark.parametrize("kernel", [P.DEEP, P.SHALLOW])
def test_fused_loop_over_many_steps_equals_convect_plus_advance(ctx, kernel):
    """More steps than the loop's check interval (16): the fused steps (state
    advanced in place by the kernels, guard-band patches applied to the
    state) equal convect + host advance bit for bit."""
    s, T, q = G.make_config("c4", shape=(48, 96), seed=23)
    T1, q1 = T.copy(), q.copy()
    for _ in range(35):
        deep, sh = ctx.convect(s, T1, q1, kernels=kernel)
        o = deep if kernel == P.DEEP else sh
        T1 = T1 + o.tend_T
        q1 = q1 + o.tend_q
    T2, q2 = ctx.timestep(s, T, q, kernel=kernel, n_steps=35)
    assert np.array_equal(T1, T2) and np.array_equal(q1, q2)


def test_fused_loop_checks_untouched_columns_at_step_0(ctx):
    """A NaN in a column the deep kernel leaves alone (s <= threshold): the
    reference's check_finite fails after step 0's advance (T + 0 = NaN)."""
    s, T, q = G.make_config("c1", n=512, seed=4)
    cold = int(np.nonzero(s <= 0.5)[0][3])
    T = T.copy()
    T[7, cold] = np.nan
    with pytest.raises(P.ValidationError) as e:
        ctx.timestep(s, T, q, kernel=P.DEEP, n_steps=20)
    assert "step 0" in str(e.value)


def test_timestep_matches_oracle_loop(ctx):
    s, T, q = G.make_config("c2", n=2000, seed=5)
    T1, q1 = T.copy(), q.copy()
    for _ in range(3):
        od = O.convection("deep", s, T1, q1)
        T1, q1 = T1 + od.tend_T, q1 + od.tend_q
    T2, q2 = ctx.timestep(s, T, q, kernel=P.DEEP, n_steps=3)
    assert np.all(np.abs(T2 - T1) <= 1e-10 * np.abs(T1))
    assert np.all(np.abs(q2 - q1) <= np.maximum(1e-10 * np.abs(q1), 1e-14))


def test_timestep_kernel_failure_and_divergence(ctx):
    s, T, q = O.make_grid(16, 30, 1.0, 42)
    T[2, 5] = np.nan
    with pytest.raises(P.KernelError) as e:
        ctx.timestep(s, T, q, kernel=P.DEEP, n_steps=2)
    assert "column 5" in str(e.value)
    # shallow propagates NaN T into the state: check_finite fails at step 0
    with pytest.raises(P.ValidationError) as e:
        ctx.timestep(s, T, q, kernel=P.SHALLOW, n_steps=2)
    assert "step 0" in str(e.value)


def test_error_growth_identical_paths_zero_deviation(ctx):
    # acceptance.cpp:574-593: execution-order changes give zero deviation
    s, T, q = O.make_grid(64, 30, 0.3, 42)
    g = ctx.error_growth(s, T, q, P.DEEP, P.KernelOptions(), P.KernelOptions(), 50)
    assert (g.rms_mod == 0.0).all() and g.envelope_ok and g.worst_ratio == 0.0
    assert (g.rms_pert > 0.0).all()


@pytest.mark.parametrize("mod", [P.Variant.STRENGTH_REDUCED, P.Variant.APPROX_TRANSCENDENTAL])
def test_error_growth_variant_envelope_matches_reference(ctx, mod):
    # acceptance.cpp:595-613 (c11): answer-changing variants stay inside the
    # one-ulp perturbation envelope, on the device as in the reference
    s, T, q = O.make_grid(64, 30, 0.3, 42)
    ref = O.ref_error_growth("deep", s, T, q, O.EXACT, int(mod), 50)
    assert ref.status == 0
    g = ctx.error_growth(s, T, q, P.DEEP, P.KernelOptions(), P.KernelOptions(variant=mod), 50)
    assert g.envelope_ok == ref.envelope_ok and g.envelope_ok
    assert g.rms_pert[-1] > 0.0
    # the perturbation envelope grows like the reference's (a chaotic map:
    # same order of magnitude at every step, not the same bits)
    ratio = g.rms_pert / ref.rms_pert
    assert (ratio > 0.1).all() and (ratio < 10.0).all()


def test_relaxed_update_inside_rounding_envelope(ctx):
    """The relaxed Newton update (default for Exact) against the strict,
    reference-rounding update: the paper's acceptance test for an
    answer-changing optimisation -- its deviation must stay inside the
    one-ulp perturbation envelope."""
    s, T, q = G.make_config("c1", n=512, seed=31)
    g = ctx.error_growth(s, T, q, P.DEEP, P.KernelOptions(strict=True), P.KernelOptions(), 50)
    assert g.envelope_ok, g.worst_ratio
    assert g.rms_pert[-1] > 0.0


def test_error_growth_shallow_and_rms_restatement(ctx):
    s, T, q = O.make_grid(96, 30, 0.3, 7)
    g = ctx.error_growth(s, T, q, P.SHALLOW, P.KernelOptions(), P.KernelOptions(variant=2), 5)
    ref = O.ref_error_growth("shallow", s, T, q, O.EXACT, O.APPROX_TRANSCENDENTAL, 5)
    assert g.envelope_ok == ref.envelope_ok
    # rms_pert after one step, restated on the host from the device's own legs
    Tb, _ = ctx.timestep(s, T, q, kernel=P.SHALLOW, n_steps=1)
    Tp0 = (T.view(np.int64) ^ 1).view(np.float64)
    Tp, _ = ctx.timestep(s, Tp0, q, kernel=P.SHALLOW, n_steps=1)
    assert abs(g.rms_pert[0] - host_rms(Tp, Tb)) <= 1e-12 * host_rms(Tp, Tb)


def test_error_growth_rejects_non_finite_initial_state(ctx):
    s, T, q = O.make_grid(8, 30, 0.3, 1)
    T[3, 2] = np.inf
    with pytest.raises(P.ValidationError) as e:
        ctx.error_growth(s, T, q, P.DEEP, timesteps=3)
    assert "perturb_lsb" in str(e.value)
