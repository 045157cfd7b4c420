"""The package exports every public name of the reference's ``adrom``
package (/root/reference/pkg/src/adrom/__init__.py:6-66), so a user of the
reference finds the same API surface (list frozen here; the reference tree
is not read at test time)."""

REFERENCE_EXPORTS = """
NewtonResult SvdResult least_squares newton_solve orth pivoted_qr principal_angles thin_svd
ExperimentConfig RunResult acceleration make_problem relative_error run_adaptive_rom run_fom
run_static_rom BurgersProblem SodProblem TimeStepper coarse_step fd_jacobian implicit_step
rusanov_flux sod_initial_state ReducedState RomOperator build_rom_operator decode encode
galerkin_step lspg_objective lspg_step rom_step FeatureMap SamplingSet build_deim_operator
fgs_sample qdeim_sample stencil_closure ScalingTransform fit_scaling pod ReducedBasis
SnapshotWindow UpdateRule direct_update grouse_update isvd_update oja_update onestep_update
wsvd_update
""".split()


def test_reference_names_exported():
    import paper_2605_28684_b200 as P
    missing = [n for n in REFERENCE_EXPORTS if not hasattr(P, n)]
    assert not missing, missing


def test_update_rule_validation():
    import pytest
    from paper_2605_28684_b200 import SnapshotWindow, UpdateRule
    with pytest.raises(ValueError):
        UpdateRule("sgd")
    with pytest.raises(ValueError):
        UpdateRule("isvd", lam=1.5)
    with pytest.raises(ValueError):
        UpdateRule("oja", eta=0.0)
    with pytest.raises(ValueError):
        UpdateRule("wsvd", window=0)
    with pytest.raises(ValueError):
        SnapshotWindow(0)
    assert UpdateRule("wsvd", window=3).label() == "wsvd(w=3)"
    assert UpdateRule("grouse", eta=0.5).label() == "grouse(eta=0.5)"
    assert UpdateRule("direct").uses_window and not UpdateRule("oja").history_aware
