"""CPU: pin the oracle (a numpy restatement of the reference) to the reference's
own outputs (tests/golden, produced by importing /root/reference) and to the
known answers in the reference's tests. Also pins the product's geometry types
(fingerprints and voxel centres) to the reference."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, rc, rel_l2, small, tiny
from oracle import nfmimo_oracle as O
from paper_2509_00774_b200 import configs


def test_known_answers_direct_formula():
    ka = golden("known_answers")
    c = 299_792_458.0

    def elem(tx, rx, vox, f):
        g = O.Geom(np.array([tx], float), np.array([rx], float), np.array([f]), np.array([1 + 0j]),
                   np.array([vox], float), c)
        return O.element_row(g, 0)[0]

    # GOLDEN_ELEMENT, test_forward.py:26-28, 54-62
    assert elem((0.1, 0, 0), (-0.1, 0, 0), (0, 0, 0.4), 10e9) == pytest.approx(
        -0.4677243613935091 + 0.018818304865202827j, rel=1e-13)
    assert elem((0.1, 0, 0), (-0.1, 0, 0), (0, 0, 0.4), 10e9) == pytest.approx(complex(ka["golden_element"]), rel=1e-14)
    # full wave → 1/π, quarter wave → −j/π (test_forward.py:43-52)
    assert elem((0, 0, 0), (0, 0, 0), (0, 0, 0.5), c) == pytest.approx(1 / np.pi, rel=1e-12)
    assert elem((0, 0, 0), (0, 0, 0), (0, 0, 0.5), c / 4) == pytest.approx(-1j / np.pi, rel=1e-12)


def test_soft_threshold_and_change_known_answers():
    ka = golden("known_answers")
    assert O.soft_threshold(ka["soft_in"], float(ka["soft_alpha"]))[0] == pytest.approx(1.8 + 2.4j, rel=1e-15)
    assert np.array_equal(O.soft_threshold(ka["soft_in"], float(ka["soft_alpha"])), ka["soft_out"])
    assert np.array_equal(O.soft_threshold(np.array([0.5 + 0.5j, -0.1j, 0j]), 1.0), np.zeros(3))
    assert O.relative_magnitude_change(np.array([1.0 + 0j, 0.0]), np.array([1.1 + 0j, 0.0])) == pytest.approx(
        float(ka["change"]), rel=1e-15)
    with pytest.raises(ValueError):
        O.soft_threshold(np.array([1.0 + 0j]), -0.1)


@pytest.mark.parametrize("name,builder", [("tiny", tiny), ("small", small)])
def test_geometry_fingerprint_matches_reference(name, builder):
    g = golden("unit_scenarios")
    from paper_2509_00774_b200.geometry import scenario_fingerprint

    assert scenario_fingerprint(builder()) == bytes(g[f"{name}_fingerprint"])


@pytest.mark.parametrize("name,builder", [("tiny", tiny), ("small", small)])
def test_oracle_matches_reference_dense_and_ops(name, builder):
    g = golden("unit_scenarios")
    geo = O.geom_from_scenario(builder())
    dense = np.stack([O.element_row(geo, m) for m in range(geo.M)])
    assert np.allclose(dense, g[f"{name}_dense"], rtol=1e-13, atol=0)
    op = O.TableOperator(geo)
    s, r, sub = g[f"{name}_s"], g[f"{name}_r"], g[f"{name}_sub"]
    # the table restatement reproduces the reference bit for bit
    assert np.array_equal(op.forward(s, np.arange(geo.M)), g[f"{name}_fwd"])
    assert np.array_equal(op.forward(s, sub), g[f"{name}_fwd_sub"])
    assert rel_l2(op.adjoint(r, np.arange(geo.M)), g[f"{name}_adj"]) <= 1e-15
    assert rel_l2(op.adjoint(r[: sub.size], sub), g[f"{name}_adj_sub"]) <= 1e-15
    # the direct formula agrees to rounding
    assert rel_l2(O.direct_forward(geo, s, np.arange(geo.M)), g[f"{name}_fwd"]) <= 1e-13
    assert rel_l2(O.direct_adjoint(geo, r, np.arange(geo.M)), g[f"{name}_adj"]) <= 1e-13


def test_oracle_lipschitz_and_structured_spgm_match_reference():
    g = golden("unit_scenarios")
    geo = O.geom_from_scenario(small())
    op = O.TableOperator(geo)
    assert O.lipschitz(op, n_iters=500, tol=1e-13) == pytest.approx(float(g["small_lipschitz"]), rel=1e-12)
    # replay the reference's structured SPGM with the oracle loop and the reference sampler's
    # index sequence (recomputed with the same numpy calls, solver.py:206-225)
    rng = np.random.default_rng(9)
    seq = []
    F, T, R = geo.F, geo.T, geo.R
    for _ in range(30):
        fs = np.sort(rng.choice(F, 2, replace=False))
        ts = np.sort(rng.choice(T, 2, replace=False))
        rs = np.sort(rng.choice(R, 1, replace=False))
        seq.append((rs[None, None, :] + R * (ts[None, :, None] + T * fs[:, None, None])).reshape(-1))
    assert np.array_equal(seq[0], g["small_structured_first_batch"])
    s, changes = O.spgm(op, g["small_y"], 1e-3, 4e-5, seq)
    assert rel_l2(s, g["small_spgm_structured"]) <= 1e-13
    assert np.allclose(changes, g["small_spgm_changes"], rtol=1e-10)


def test_oracle_replays_baseline_small():
    """BASELINE config 0 (Small): scene, noise, L, λ and 200 flat SPGM iterations."""
    b = golden("baseline_small")
    w = configs.WORKLOADS["small"]()
    from paper_2509_00774_b200.geometry import scenario_fingerprint

    assert scenario_fingerprint(w.scenario) == bytes(b["fingerprint"])
    assert np.array_equal(configs.make_scene(w), b["s_true"])
    geo = O.geom_from_scenario(w.scenario)
    op = O.TableOperator(geo)
    clean = op.forward(b["s_true"], np.arange(geo.M))
    assert rel_l2(clean, b["clean"]) <= 1e-15
    assert configs.noise_sigma(clean, w.snr_db) == pytest.approx(float(b["sigma"]), rel=1e-14)
    assert rel_l2(configs.add_noise(clean, float(b["sigma"])), b["y"]) <= 1e-15
    assert O.lipschitz(op, n_iters=20) == pytest.approx(float(b["L"]), rel=1e-12)
    seq = O.flat_index_sequence(geo.M, w.batch, w.iters, configs.SEEDS["minibatch"])
    assert np.array_equal(np.stack(seq), b["index_table"])
    s, changes = O.spgm(op, b["y"], float(b["eta"]), float(b["alpha"]), seq)
    assert rel_l2(s, b["s_final"]) <= 1e-12
    assert np.allclose(changes, b["changes"], rtol=1e-9)


def test_oracle_direct_formula_matches_reference_medium():
    """BASELINE config 1 (Medium): the reference's cached-table outputs vs the table-free oracle."""
    m = golden("medium_ops")
    w = configs.WORKLOADS["medium"]()
    geo = O.geom_from_scenario(w.scenario)
    s = rc(np.random.default_rng(int(m["s_seed"])), geo.N)
    r = rc(np.random.default_rng(int(m["r_seed"])), m["idx"].size)
    assert rel_l2(O.direct_forward(geo, s, m["idx"]), m["fwd"]) <= 1e-12
    probe = m["adj_probe_voxels"][:1024]
    assert rel_l2(O.direct_adjoint(geo, r, m["idx"], voxels=probe), m["adj_probe"][:1024]) <= 1e-12


def test_flat_sequence_is_sorted_distinct():
    seq = O.flat_index_sequence(1000, 64, 5, 0)
    for idx in seq:
        assert np.all(np.diff(idx) > 0) and idx.min() >= 0 and idx.max() < 1000


@pytest.mark.parametrize("name", ["tiny", "ragged"])
def test_oracle_with_tabulated_pulse_matches_reference(name):
    """The oracle's table restatement and direct formula carry p(f) as the reference does (p_f in the
    forward, forward.py:283-284; conj p_f in the adjoint, :315-325): bit-exact table restatement and
    1e-12 direct formula against the reference's outputs (tests/golden/pulse_scenarios.npz)."""
    import pulse_cases
    from paper_2509_00774_b200.geometry import scenario_fingerprint

    g = golden("pulse_scenarios")
    scn = pulse_cases.CASES[name]()
    assert scenario_fingerprint(scn) == bytes(g[f"{name}_fingerprint"])
    geo = O.geom_from_scenario(scn)
    assert np.ptp(np.angle(geo.pulse)) > 0.1  # genuinely frequency dependent and complex
    s, r, sub = g[f"{name}_s"], g[f"{name}_r"], g[f"{name}_sub"]
    op = O.TableOperator(geo)
    full = np.arange(geo.M)
    assert np.array_equal(op.forward(s, full), g[f"{name}_fwd"])
    assert np.array_equal(op.forward(s, sub), g[f"{name}_fwd_sub"])
    assert rel_l2(op.adjoint(r, full), g[f"{name}_adj"]) <= 1e-14
    assert rel_l2(O.direct_forward(geo, s, full), g[f"{name}_fwd"]) <= 1e-12
    assert rel_l2(O.direct_adjoint(geo, r[: sub.size], sub), g[f"{name}_adj_sub"]) <= 1e-12


def test_baseline_medium_fixture_is_the_reference_sampler():
    """The Medium reconstruction fixture (reference run, make_golden.py gen_baseline_medium): its index
    table is the reference sampler's numpy call sequence, as the oracle restates it, and its step size
    and threshold follow the BASELINE recipe (eta = 1/L, alpha = eta * 1e-3 max|A^H y| / M)."""
    b = golden("baseline_medium")
    w = configs.WORKLOADS["medium"]()
    M = w.scenario.n_channels
    table = np.stack(O.flat_index_sequence(M, w.batch, w.iters, configs.SEEDS["minibatch"]))
    assert np.array_equal(table, b["index_table"])
    assert float(b["eta"]) == pytest.approx(1.0 / float(b["L"]), rel=1e-15)
    assert float(b["alpha"]) == pytest.approx(float(b["eta"]) * float(b["lam"]), rel=1e-15)
    assert b["s_final"].shape == (w.scenario.n_voxels,) and b["changes"].shape == (w.iters,)


def test_paper_v_fixture_matches_recorded_reference_run():
    """The paper-v study fixture agrees with the reference's own recorded acceptance run
    (pkg/test_output.txt:221-225): PGM converges in 590 iterations, SPGM(4,4,3) PSNR 44.9 / 45.0 /
    45.4 dB for seeds 1-3, argmax voxel 70010."""
    g = golden("paper_v_study")
    assert int(g["pgm_iterations"]) == 590
    assert [round(float(g[f"spgm{k}_psnr"]), 1) for k in (1, 2, 3)] == [44.9, 45.0, 45.4]
    assert int(g["loc_found_voxel"]) == int(g["loc_true_voxel"]) == 70010
