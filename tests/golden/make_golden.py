"""Generate tests/golden/tfhe_golden_seed42.npz (CGGI key layout, bk_unroll 1)
and tests/golden/tfhe_golden_pairs_seed42.npz (key-pair layout, bk_unroll 2)
with the CPU oracle.

The reference ships no TFHE code or known-answer ciphertexts, so these vectors
pin the oracle restatement against later changes (and the GPU engine against
the oracle); they are not reference outputs.  Run:  python tests/golden/make_golden.py
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402



def make(unroll, name):
    P = O.default_params()
    P.bk_unroll = unroll
    keys = O.Keys(P, 42)
    ctx = O.Context(P, keys)
    bits = np.array([1, 0, 1, 1, 0, 0, 1, 0], np.uint8)
    inputs = O.encrypt(P, keys, bits, 42, 77)
    rng = np.random.default_rng(42)
    ks_in = rng.integers(0, 2 ** 32, P.N + 1, dtype=np.uint64).astype(np.uint32)
    out = {
        "lwe_key": keys.lwe_key,
        "bk_sum": np.uint64(keys.bk.astype(np.uint64).sum()),
        "ksk_sum": np.uint64(keys.ksk.astype(np.uint64).sum()),
        "input_bits": bits,
        "inputs": inputs,
        # CGGI: 3 key bits; key pairs: 2 pairs (4 key bits)
        "acc_prefix3": ctx.blind_rotate(inputs[0], iters=3 if unroll == 1 else 4),
        "bootstrap_wo_ks": ctx.bootstrap_wo_ks(inputs[2]),
        "ks_in": ks_in,
        "ks_out": ctx.keyswitch(ks_in),
    }
    for gname, (c0, al, be) in O.GATE_LIN.items():
        out[f"gate_{gname}"] = ctx.gate(c0, al, inputs[0], be, inputs[1])
    out["mux_010"] = ctx.mux(inputs[1], inputs[0], inputs[4])  # s=0 -> selects third
    out["mux_110"] = ctx.mux(inputs[0], inputs[2], inputs[1])  # s=1 -> selects second
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), name)
    np.savez_compressed(path, **out)
    print("wrote", path)


if __name__ == "__main__":
    make(1, "tfhe_golden_seed42.npz")
    make(2, "tfhe_golden_pairs_seed42.npz")
