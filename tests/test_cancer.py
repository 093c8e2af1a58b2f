"""The reference's shipped Cancer model on the reference's own dataset rows
(VERDICT r1 f4): the binned fixture (tests/golden/make_cancer_fixture.py) is
pinned by reproducing the trainer's reported accuracies exactly through
oracle_eval, and the encrypted classification (lanes) matches oracle_eval row
by row on the stand-in engine here and on the B200 (test_gpu_cancer)."""

import numpy as np
import pytest

from hebnn.model import oracle_eval
from paper_1806_03461_b200 import workloads
from plain_engine import plain_context_class


def test_fixture_reproduces_the_trainer_accuracies():
    X, y, train, test, (acc_train, acc_test) = workloads.cancer_rows()
    assert X.shape == (569, 90) and set(np.unique(X)) <= {0, 1}
    assert (X.reshape(569, 30, 3).sum(axis=2) == 1).all()  # one hot bin per feature
    assert len(train) == 398 and len(test) == 171
    assert sorted(np.concatenate([train, test]).tolist()) == list(range(569))
    model = workloads.cancer_model()
    pred = np.array([oracle_eval(model, [1 if v else -1 for v in row])[0] for row in X])
    assert (pred[train] == y[train]).mean() == acc_train  # 0.9597989949748744 (metrics.json)
    assert (pred[test] == y[test]).mean() == acc_test     # 0.9649122807017544


def test_encrypted_lanes_match_oracle_on_plain_engine():
    rep = workloads.run_cancer(plain_context_class(), rows=np.arange(0, 569, 7))
    assert rep["matches_oracle_eval"] is True


@pytest.mark.gpu
def test_gpu_cancer_all_rows():
    """All 569 rows encrypted, one DAG with 569 lanes, on the B200."""
    from paper_1806_03461_b200.backend import TfheContext

    rep = workloads.run_cancer(TfheContext)
    assert rep["matches_oracle_eval"] is True
    assert rep["accuracy_test"] == rep["trainer_accuracy"]["test"]
    assert rep["accuracy_train"] == rep["trainer_accuracy"]["train"]
