"""f3/f4 on the GPU: the reference CLI running on the B200 backend, and the
client/server split with serialised evaluation keys and ciphertexts."""

import json
import os

import numpy as np
import pytest

from paper_1806_03461_b200 import cli, wire_keys
from paper_1806_03461_b200.backend import TfheContext
from paper_1806_03461_b200.tfhe import KeySet

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
MODEL = os.path.join(HERE, "golden", "cancer_model.json")


def test_cli_eval_on_b200_equals_simulator(tmp_path, capsys):
    inp = tmp_path / "x.json"
    inp.write_text(json.dumps({"version": 1, "encoding": "pm1", "values": [1, 1, -1] * 30}))
    assert cli.main(["--backend", "sim", "eval", "--model", MODEL, "--input", str(inp)]) == 0
    want = json.loads(capsys.readouterr().out)
    assert cli.main(["--backend", "tfhe-b200", "--key-seed", "42", "eval", "--model", MODEL, "--input", str(inp)]) == 0
    got = json.loads(capsys.readouterr().out)
    assert got == want  # prediction and (data-oblivious) estimates identical


def test_cli_calibrate_and_b200_estimate(capsys):
    assert cli.main(["calibrate"]) == 0
    cal = json.loads(capsys.readouterr().out)
    assert 0 < cal["t_gate_s"] < 0.1 and cal["intra_workers"] >= 4 * 100
    assert cli.main(["estimate", "--model", MODEL, "--t-gate", "b200"]) == 0
    rep = json.loads(capsys.readouterr().out)
    assert rep["estimates"]["out_seq"] < 1.0  # the paper's 3.5 s Cancer estimate at 0.1 s/gate


def test_client_server_split(tmp_path):
    from hebnn.compiler import eval_model
    from hebnn.model import oracle_eval
    from hebnn.wire import parse_model

    model = parse_model(json.load(open(MODEL)))
    client = KeySet(seed=99)
    wire_keys.save_keys(tmp_path / "ek.npz", client)
    xs = [1, -1, -1] * 30
    wire_keys.save_ciphertexts(tmp_path / "in.npz", client.encrypt([1 if v == 1 else 0 for v in xs], seed=5),
                               client.params)
    # server: evaluation keys + encrypted input only
    server_keys = wire_keys.load_keys(tmp_path / "ek.npz")
    cts, _ = wire_keys.load_ciphertexts(tmp_path / "in.npz")
    ctx = TfheContext(keys=server_keys)
    outs, _ = eval_model(ctx, model, ctx.import_ciphertexts(cts))
    with pytest.raises(PermissionError):
        ctx.decrypt(outs[0])
    wire_keys.save_ciphertexts(tmp_path / "out.npz", ctx.export_ciphertexts(outs)[:, 0, :], server_keys.params)
    # client decrypts
    res, _ = wire_keys.load_ciphertexts(tmp_path / "out.npz")
    pred = [1 if b else -1 for b in client.decrypt(res)]
    assert pred == oracle_eval(model, xs)
