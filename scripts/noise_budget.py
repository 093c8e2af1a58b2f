"""Noise budget of the parameter set (BASELINE.json configs[0]) and the
resulting decryption-failure probability, using the standard CGGI variance
propagation (independent uniform digits, binary keys), for both
bootstrapping-key layouts:
  bk_unroll 1 (CGGI): n external products, TGSW noise sigma_bk each;
  bk_unroll 2 (key pairs): n/2 external products with the combined TGSW
    sum_c (X^e_c - 1) BK_c: 3 components x 2 monomials = 6 noise terms per
    coefficient (3x the BK variance of the CGGI key over the whole rotation),
    and half the gadget-rounding terms.
Prints the table used in DESIGN.md §Parameters."""

import math

n, N, k, bg_bits, l, ks_bits, ks_t = 630, 1024, 1, 7, 3, 2, 8
s_lwe, s_bk = 2.0 ** -15, 2.0 ** -25
Bg = 2 ** bg_bits
var_digit = (Bg ** 2 - 1) / 12.0                       # uniform digits in [-Bg/2, Bg/2)
eps = 1.0 / (2 * Bg ** l)                               # gadget precision


def budget(unroll):
    bk_terms, round_terms = (n, n) if unroll == 1 else (3 * n, n // 2)
    var_br = bk_terms * (k + 1) * l * N * var_digit * s_bk ** 2   # BK noise through the external products
    var_br += round_terms * (1 + k * N) * eps ** 2 / 3 * 0.5      # decomposition rounding (binary key)
    var_ks = k * N * ks_t * s_lwe ** 2                            # KSK noise
    var_ks += k * N * (2.0 ** -(ks_bits * ks_t + 1)) ** 2 / 3 * 0.5
    return var_br, var_ks


def sigma_out(unroll):
    var_br, var_ks = budget(unroll)
    return math.sqrt(var_br + var_ks)


if __name__ == "__main__":
    var_ms = (n * 0.5 + 1) * (1.0 / (4 * N)) ** 2 / 3       # mod switch to Z_2N
    for unroll in (1, 2):
        var_br, var_ks = budget(unroll)
        var_out = var_br + var_ks
        print(f"bk_unroll {unroll} ({'CGGI' if unroll == 1 else 'key pairs'})")
        print(f"  sigma_BR   = 2^{math.log2(math.sqrt(var_br)):.2f}")
        print(f"  sigma_KS   = 2^{math.log2(math.sqrt(var_ks)):.2f}")
        print(f"  sigma_out  = 2^{math.log2(math.sqrt(var_out)):.2f}  (gate output, torus units)")
        print(f"  sigma_ms   = 2^{math.log2(math.sqrt(var_ms)):.2f}  (mod-switch rounding)")
        for name, coef, margin in (("AND/OR/NAND/NOR (|coef| 1)", 2 * 1, 1 / 8), ("XOR/XNOR (|coef| 2)", 2 * 4, 1 / 4),
                                   ("MUX half (S +- A)", 2 * 1, 1 / 8)):
            var = coef * var_out + var_ms
            z = margin / math.sqrt(var)
            p = math.erfc(z / math.sqrt(2))
            print(f"  {name:28s} sigma = 2^{math.log2(math.sqrt(var)):.2f}  margin {margin}  z = {z:.1f}  "
                  f"P(fail) ~ 2^{math.log2(p) if p > 0 else float('-inf'):.0f}")
        # inputs produced by a plain gate (1 blind rotation + KS) or by a MUX / the XOR
        # output of a fused half adder (2 blind-rotation noise terms + 1 KS), into every
        # consumer: 2-input (|coef| 1 or 2) and 3-input (majority |coef| 1, XOR3 |coef| 2)
        var_two = 2 * var_br + var_ks
        for src, v_in in (("gate outputs", var_out), ("MUX / HA-XOR outputs", var_two)):
            for name, terms, coef2, margin in (("AND/OR", 2, 1, 1 / 8), ("XOR", 2, 4, 1 / 4),
                                               ("MAJ", 3, 1, 1 / 8), ("XOR3", 3, 4, 1 / 4)):
                var = terms * coef2 * v_in + var_ms
                z = margin / math.sqrt(var)
                p = math.erfc(z / math.sqrt(2))
                print(f"  {name:6s} of {terms} {src:22s} z = {z:5.1f}  P(fail) ~ 2^{math.log2(p) if p > 0 else float('-inf'):.0f}")
