"""Estimator facade on the CPU host: parameter protocol and argument checks
(the device queries are covered in test_gpu_parity.py)."""
import pytest

from paper_1202_3777_b200.estimator import JunctionTreeEngine


def test_params_roundtrip():
    est = JunctionTreeEngine(dtype="f32", batch=64, target="x")
    p = est.get_params()
    assert p["dtype"] == "f32" and p["batch"] == 64 and p["target"] == "x" and p["engine"] == "cuda"
    est.set_params(batch=8)
    assert est.batch == 8


@pytest.mark.parametrize("kw", [{"engine": "gpu"}, {"engine": "sequential"}, {"layout": "diagonal"}, {"batch": 0}])
def test_bad_params_raise(kw):  # the reference rejects unknown engines (test_estimator.py:28-32)
    with pytest.raises(ValueError):
        JunctionTreeEngine(**kw).fit_compiled(None, None)


def test_unfitted_raises():
    with pytest.raises(ValueError):
        JunctionTreeEngine(target="x").predict_proba([{}])
