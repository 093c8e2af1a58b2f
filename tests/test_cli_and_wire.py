"""CLI backend hook (f3) and key/ciphertext documents (f4) — host side."""

import json
import os

import numpy as np
import pytest

from paper_1806_03461_b200 import cli, wire_keys
from paper_1806_03461_b200.tfhe import KeySet

HERE = os.path.dirname(os.path.abspath(__file__))
MODEL = os.path.join(HERE, "golden", "cancer_model.json")


def test_cli_sim_backend_matches_reference_cli(tmp_path, capsys):
    inp = tmp_path / "x.json"
    inp.write_text(json.dumps({"version": 1, "encoding": "pm1", "values": [1, -1] * 45}))
    from hebnn import cli as ref_cli

    assert ref_cli.main(["eval", "--model", MODEL, "--input", str(inp)]) == 0
    want = json.loads(capsys.readouterr().out)
    assert cli.main(["--backend", "sim", "eval", "--model", MODEL, "--input", str(inp)]) == 0
    got = json.loads(capsys.readouterr().out)
    assert got == want


def test_cli_error_exit_code_preserved(tmp_path, capsys):
    assert cli.main(["--backend", "sim", "eval", "--model", str(tmp_path / "missing.json"),
                     "--input", str(tmp_path / "x.json")]) in (1, 2)


def test_key_and_ciphertext_documents_roundtrip(tmp_path, keys):
    p = tmp_path / "eval_keys.npz"
    wire_keys.save_keys(p, keys)
    server = wire_keys.load_keys(p)
    assert not server.has_secret
    assert np.array_equal(server.bk, keys.bk) and np.array_equal(server.ksk, keys.ksk)
    with pytest.raises(PermissionError):
        server.decrypt(np.zeros((1, 631), np.uint32))
    full = tmp_path / "keyset.npz"
    wire_keys.save_keys(full, keys, include_secret=True)
    client = wire_keys.load_keys(full)
    cts = client.encrypt(np.array([1, 0, 1], np.uint8), seed=4)
    c = tmp_path / "cts.npz"
    wire_keys.save_ciphertexts(c, cts, client.params, meta={"model": "cancer"})
    back, meta = wire_keys.load_ciphertexts(c)
    assert meta == {"model": "cancer"}
    assert list(keys.decrypt(back)) == [1, 0, 1]


def test_wrong_document_kind_rejected(tmp_path, keys):
    c = tmp_path / "cts.npz"
    wire_keys.save_ciphertexts(c, keys.encrypt([1], seed=1), keys.params)
    with pytest.raises(ValueError):
        wire_keys.load_keys(c)


def test_key_document_validation(tmp_path, keys):
    """A truncated or mismatched eval-key document is rejected before the engine
    would copy hb_bk_words / hb_ksk_words words from it."""
    import json as _json

    def write(path, header, **arrays):
        np.savez(path, header=np.frombuffer(_json.dumps(header).encode(), np.uint8), **arrays)

    good = tmp_path / "good.npz"
    wire_keys.save_keys(good, keys)
    with np.load(good) as z:
        hdr = _json.loads(bytes(z["header"]).decode())
        bk, ksk = z["bk"], z["ksk"]
    cases = {
        "truncated_bk": (hdr, dict(bk=bk[:-1], ksk=ksk)),
        "truncated_ksk": (hdr, dict(bk=bk, ksk=ksk[: ksk.size // 2])),
        "wrong_dtype": (hdr, dict(bk=bk.astype(np.int64), ksk=ksk)),
        "two_d": (hdr, dict(bk=bk.reshape(2, -1), ksk=ksk)),
        "missing_ksk": (hdr, dict(bk=bk)),
        "params_mismatch": ({**hdr, "params": {**hdr["params"], "n": 500}}, dict(bk=bk, ksk=ksk)),
        "unsupported_n": ({**hdr, "params": {**hdr["params"], "n": 750}}, dict(bk=bk, ksk=ksk)),
        "bad_params": ({**hdr, "params": {"n": 630}}, dict(bk=bk, ksk=ksk)),
    }
    for name, (h, arrays) in cases.items():
        p = tmp_path / f"{name}.npz"
        write(p, h, **arrays)
        with pytest.raises(ValueError):
            wire_keys.load_keys(p)
    assert wire_keys.load_keys(good).bk.size == bk.size
