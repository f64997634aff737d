"""B200 re-calibration artefacts (tools/calibrate.py output) in the reference's schemas."""
import json
import pathlib

from paper_2512_10236_b200 import machines, pricing, selector
from paper_2512_10236_b200.ops import _scenario

ROOT = pathlib.Path(__file__).resolve().parents[1]
DATA = ROOT / "paper_2512_10236_b200" / "data"


def test_calibration_file_passes_reference_validation():
    doc = json.loads((DATA / "calibration_b200.json").read_text())
    doc.pop("_comment", None)
    model = pricing.load_calibration(json.dumps(doc))  # trend / dominance / >= 1 rules (lossmodel.py:153-179)
    assert set(model.gemm_dil_tables) == {"row8", "row64", "col8", "col64"}


def test_b200_machine_file_loads_with_fitted_t_ref():
    spec = machines.b200_machine()
    assert spec.topo.kind.value == "switch" and spec.topo.n_gpus == 8
    assert 0 < spec.t_ref < 1.0  # re-fitted: the reference default 1.0 s sends every sub-second GEMM to uniform


def test_fitted_selector_reproduces_recorded_agreement():
    """The selector with the fitted t_ref picks the measured-best fine-grain schedule as often as
    the calibration run recorded (profiles/r01_calibration.json)."""
    rec = json.loads((ROOT / "profiles" / "r01_calibration.json").read_text())
    spec = machines.b200_machine()
    ok = 0
    for row in rec["scenarios"]:
        m, n, k = row["scenario"]
        valid = {kk: v for kk, v in row["kinds_s"].items() if v}
        best = min(valid, key=valid.get)
        ok += selector.select_schedule(_scenario("x", m, n, k, 8), spec.machine, spec.t_ref).value == best
    assert ok == rec["heuristic_agreement"][0]
    # The selector's shape (uniform for small 2MNK, hetero_fused in between, hetero_unfused for large)
    # does not match what wins on this executor (hetero_unfused already wins small shapes), and
    # kinds are often within a few % of each other, so the measured best flips between boxes: 9/10
    # on the first calibration pod, 6/10 on the current one. Bound the agreement and the regret.
    assert ok / len(rec["scenarios"]) >= 0.6
    assert rec["mean_regret_on_mismatches"] <= 0.15


def test_b200_calibration_loads_through_the_strict_loader():
    from paper_2512_10236_b200 import machines, pricing
    model = machines.b200_calibration()
    assert isinstance(model, pricing.LossModel)
