"""Device-resident ciphertext exchange (hb_pool_gather_device /
hb_pool_put_device): export to / import from CUDA tensors without host
staging, and Out-P layers chained through it (single rank, identity
all-gather) — decrypted scores equal oracle_eval."""

import random

import numpy as np
import pytest

from hebnn.model import DenseLayer, SignActivation, TernaryModel, oracle_eval, validate_model

pytestmark = pytest.mark.gpu


def test_export_import_device_roundtrip():
    from paper_1806_03461_b200.backend import TfheContext

    a = TfheContext(seed=42, enc_stream=5)
    bits = [a.encrypt(v) for v in (1, 0, 1, 1)]
    outs = [a.g_and(bits[0], bits[1]), a.g_not(a.g_xor(bits[2], bits[3])), a.trivial_const(1), bits[0]]
    dev = a.export_ciphertexts_device(outs)
    host = a.export_ciphertexts(outs)
    assert np.array_equal(dev.cpu().numpy().view(np.uint32), host)
    b = TfheContext(seed=42, enc_stream=6)
    got = [b.decrypt(h) for h in b.import_ciphertexts_device(dev)]
    assert got == [0, 1, 1, 1]


class _LocalDeviceComm:
    rank, world, device_tensors = 0, 1, True

    def all_gather(self, arr):
        return [arr]

    def all_gather_tensor(self, t):
        return [t]


def test_outp_layers_chained_on_device():
    from paper_1806_03461_b200.backend import TfheContext, shared_keys
    from paper_1806_03461_b200.parallel import OutPEvaluator, decode_scores

    rng = random.Random(5)
    d, h, p = 48, 7, 3
    l1 = tuple(tuple(rng.choice((-1, 1)) for _ in range(d)) for _ in range(h))
    l2 = tuple(tuple(rng.choice((-1, 0, 1)) for _ in range(h)) for _ in range(p))
    model = validate_model(TernaryModel(d, (DenseLayer(l1, (0,) * h), SignActivation(),
                                            DenseLayer(l2, (1,) * p)), "score_words"))
    xs = [rng.choice((-1, 1)) for _ in range(d)]
    cts = shared_keys(42).encrypt(np.array([1 if v == 1 else 0 for v in xs], np.uint8), seed=8, stream=3)
    ev = OutPEvaluator(lambda: TfheContext(seed=42), _LocalDeviceComm())
    words = ev.run(model, cts[:, None, :])
    scores = [int(v) for v in decode_scores(TfheContext(seed=42), words)[0]]
    assert scores == oracle_eval(model, xs)
