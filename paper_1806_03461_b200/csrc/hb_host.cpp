// Host side of the engine: parameters, deterministic ChaCha20 streams, key
// generation, encryption and decryption.  These replace the plaintext store of
// the reference's SimContext (backend.py:171-190): `encrypt` returns a real
// LWE sample, `decrypt` computes its phase.  Multi-threaded with std::thread;
// bit-identical to the oracle restatement (tests/test_oracle.py).
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "hb_internal.h"

namespace hb {

thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

// ---- ChaCha20 -------------------------------------------

static inline uint32_t rotl(uint32_t a, int b) { return (a << b) | (a >> (32 - b)); }

static inline void quarter(uint32_t &a, uint32_t &b, uint32_t &c, uint32_t &d) {
    a += b; d ^= a; d = rotl(d, 16);
    c += d; b ^= c; b = rotl(b, 12);
    a += b; d ^= a; d = rotl(d, 8);
    c += d; b ^= c; b = rotl(b, 7);
}

void chacha_block(const uint32_t key[8], uint64_t nonce, uint64_t counter, uint32_t out[16]) {
    uint32_t s[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u};
    for (int i = 0; i < 8; i++) s[4 + i] = key[i];
    s[12] = (uint32_t)counter;
    s[13] = (uint32_t)(counter >> 32);
    s[14] = (uint32_t)nonce;
    s[15] = (uint32_t)(nonce >> 32);
    uint32_t x[16];
    std::memcpy(x, s, sizeof x);
    for (int r = 0; r < 10; r++) {
        quarter(x[0], x[4], x[8], x[12]);
        quarter(x[1], x[5], x[9], x[13]);
        quarter(x[2], x[6], x[10], x[14]);
        quarter(x[3], x[7], x[11], x[15]);
        quarter(x[0], x[5], x[10], x[15]);
        quarter(x[1], x[6], x[11], x[12]);
        quarter(x[2], x[7], x[8], x[13]);
        quarter(x[3], x[4], x[9], x[14]);
    }
    for (int i = 0; i < 16; i++) out[i] = x[i] + s[i];
}

struct Stream {
    uint32_t key[8];
    uint64_t nonce, counter = 0;
    uint32_t buf[16];
    int pos = 16;

    Stream(uint64_t seed, uint64_t nonce_) : nonce(nonce_) {
        uint64_t z = seed;
        for (int i = 0; i < 4; i++) {  // splitmix64 key expansion
            z += 0x9E3779B97F4A7C15ull;
            uint64_t t = z;
            t = (t ^ (t >> 30)) * 0xBF58476D1CE4E5B9ull;
            t = (t ^ (t >> 27)) * 0x94D049BB133111EBull;
            t ^= t >> 31;
            key[2 * i] = (uint32_t)t;
            key[2 * i + 1] = (uint32_t)(t >> 32);
        }
    }
    uint32_t u32() {
        if (pos == 16) {
            chacha_block(key, nonce, counter++, buf);
            pos = 0;
        }
        return buf[pos++];
    }
    uint64_t u64() {
        uint64_t lo = u32();
        uint64_t hi = u32();
        return lo | (hi << 32);
    }
    // Box-Muller, cosine branch, rounded onto the 2^32 torus.
    uint32_t gauss_torus(double stdev) {
        double u1 = (double)((u64() >> 11) + 1) * (1.0 / 9007199254740992.0);
        double u2 = (double)(u64() >> 11) * (1.0 / 9007199254740992.0);
        double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
        double scale = stdev * 4294967296.0;
        double v = z * scale;
        return (uint32_t)(int64_t)std::llround(v);
    }
};

enum : uint64_t { DOM_LWE_KEY = 1, DOM_TRLWE_KEY = 2, DOM_BK = 3, DOM_KSK = 4, DOM_ENC = 5, DOM_BK2 = 6 };

static inline uint32_t lwe_dot(const uint32_t *a, const uint32_t *key, int n) {
    uint32_t acc = 0;
    for (int i = 0; i < n; i++) acc += a[i] & (0u - key[i]);
    return acc;
}

template <typename F>
static void parallel_for(size_t count, int threads, F &&fn) {
    if (threads <= 0) threads = (int)std::thread::hardware_concurrency();
    if (threads < 1) threads = 1;
    if ((size_t)threads > count) threads = (int)(count ? count : 1);
    if (threads == 1) {
        for (size_t i = 0; i < count; i++) fn(i);
        return;
    }
    std::vector<std::thread> pool;
    pool.reserve(threads);
    for (int t = 0; t < threads; t++) {
        pool.emplace_back([&, t]() {
            for (size_t i = (size_t)t; i < count; i += (size_t)threads) fn(i);
        });
    }
    for (auto &th : pool) th.join();
}

bool params_ok(const hb_params *p) {
    // n + 1 <= kKskStride: the device KSK table and k_keyswitch cover kKskStride output columns
    // (a_0..a_{n-1}, b), so a larger n would leave columns unwritten.
    return p && p->n > 0 && p->n <= kMaxKsN && p->N == kN && p->k == 1 && p->bg_bits == kBgBits &&
           p->l == kL && p->ks_base_bits == kKsBaseBits && p->ks_t == kKsT &&
           (p->bk_unroll == 0 || p->bk_unroll == 1 || (p->bk_unroll == 2 && (p->n & 1) == 0));
}

int bk_unroll(const hb_params *p) { return p->bk_unroll == 2 ? 2 : 1; }

size_t bk_tgsw_count(const hb_params *p) { return bk_unroll(p) == 2 ? (size_t)(p->n / 2) * 3 : (size_t)p->n; }

}  // namespace hb

using namespace hb;

extern "C" {

int hb_abi_version(void) { return HB_ABI_VERSION; }
int hb_params_valid(const hb_params *p) { return params_ok(p) ? 1 : 0; }

const char *hb_last_error(void) { return g_last_error.c_str(); }

void hb_default_params(hb_params *p) {
    p->n = 630;
    p->N = 1024;
    p->k = 1;
    p->bg_bits = 7;
    p->l = 3;
    p->ks_base_bits = 2;
    p->ks_t = 8;
    p->bk_unroll = 2;  // key pairs (one external product per two key bits)
    p->lwe_stdev = 1.0 / 32768.0;    // 2^-15
    p->bk_stdev = 1.0 / 33554432.0;  // 2^-25
}

size_t hb_lwe_words(const hb_params *p) { return (size_t)p->n + 1; }

size_t hb_bk_words(const hb_params *p) {
    return bk_tgsw_count(p) * (p->k + 1) * p->l * (p->k + 1) * p->N;
}

size_t hb_ksk_words(const hb_params *p) {
    return (size_t)p->k * p->N * p->ks_t * ((1u << p->ks_base_bits) - 1) * (p->n + 1);
}

int hb_keygen(const hb_params *p, uint64_t seed, uint32_t *lwe_key, uint32_t *trlwe_key,
              uint32_t *bk, uint32_t *ksk, int threads) {
    if (!params_ok(p) || !lwe_key || !trlwe_key || !bk || !ksk) {
        set_error("hb_keygen: unsupported parameters or null buffer");
        return HB_EINVAL;
    }
    const int n = p->n, N = p->N, k = p->k, l = p->l;
    const int base = 1 << p->ks_base_bits, t = p->ks_t;
    {
        Stream r(seed, DOM_LWE_KEY << 56);
        for (int i = 0; i < n; i++) lwe_key[i] = r.u32() & 1u;
    }
    {
        Stream r(seed, DOM_TRLWE_KEY << 56);
        for (int i = 0; i < k * N; i++) trlwe_key[i] = r.u32() & 1u;
    }
    // support of the binary TRLWE key, for the exact mask*key products
    std::vector<int> support;
    for (int i = 0; i < N; i++)
        if (trlwe_key[i]) support.push_back(i);

    const int rows = (k + 1) * l;
    // BK_i = TGSW(s_i): row (q, pp) = TRLWE(0) + s_i * 2^(32-(pp+1)Bgbits) on poly q.
    // bk_unroll 2: TGSW g = 3 m + comp of key pair (2m, 2m+1) encrypts
    // s_i s_j, s_i (1 - s_j), (1 - s_i) s_j for comp 0, 1, 2.
    const bool pairs = bk_unroll(p) == 2;
    parallel_for(bk_tgsw_count(p) * rows, threads, [&](size_t item) {
        const int g = (int)(item / rows), row = (int)(item % rows);
        uint32_t msg;
        uint64_t nonce;
        if (pairs) {
            const uint32_t si = lwe_key[2 * (g / 3)], sj = lwe_key[2 * (g / 3) + 1];
            const int comp = g % 3;
            msg = comp == 0 ? (si & sj) : comp == 1 ? (si & (1u - sj)) : ((1u - si) & sj);
            nonce = (DOM_BK2 << 56) | ((uint64_t)(g / 3) << 16) | ((uint64_t)comp << 8) | (uint64_t)row;
        } else {
            msg = lwe_key[g];
            nonce = (DOM_BK << 56) | ((uint64_t)g << 16) | (uint64_t)row;
        }
        uint32_t *trlwe = bk + item * (size_t)(k + 1) * N;
        uint32_t *mask = trlwe, *body = trlwe + (size_t)k * N;
        Stream r(seed, nonce);
        for (int j = 0; j < N; j++) mask[j] = r.u32();
        for (int j = 0; j < N; j++) body[j] = r.gauss_torus(p->bk_stdev);
        for (int s : support) {  // body += X^s * mask (negacyclic)
            for (int j = 0; j < N - s; j++) body[j + s] += mask[j];
            for (int j = N - s; j < N; j++) body[j + s - N] -= mask[j];
        }
        const int q = row / l, pp = row % l;
        trlwe[(size_t)q * N] += msg * (1u << (32 - (pp + 1) * p->bg_bits));
    });

    const int nin = k * N;
    parallel_for((size_t)nin * t * (base - 1), threads, [&](size_t item) {
        const int v = (int)(item % (base - 1)) + 1;
        const int j = (int)((item / (base - 1)) % t);
        const int i = (int)(item / ((size_t)(base - 1) * t));
        uint32_t *ct = ksk + item * (size_t)(n + 1);
        const uint64_t id = ((uint64_t)i * t + j) * base + v;
        Stream r(seed, (DOM_KSK << 56) | id);
        for (int a = 0; a < n; a++) ct[a] = r.u32();
        const uint32_t msg = (trlwe_key[i] * (uint32_t)v) << (32 - (j + 1) * p->ks_base_bits);
        ct[n] = lwe_dot(ct, lwe_key, n) + r.gauss_torus(p->lwe_stdev) + msg;
    });
    return HB_OK;
}

int hb_encrypt(const hb_params *p, const uint32_t *lwe_key, uint64_t seed, uint64_t stream,
               uint64_t first_index, const uint8_t *bits, size_t count, uint32_t *out, size_t out_stride) {
    if (!params_ok(p) || out_stride < (size_t)p->n + 1 || (count && (!bits || !out || !lwe_key)) ||
        first_index + count > (1ull << 32)) {
        set_error("hb_encrypt: bad arguments");
        return HB_EINVAL;
    }
    for (size_t i = 0; i < count; i++) {
        if (bits[i] > 1) {
            set_error("plaintext bit must be 0 or 1, got " + std::to_string((int)bits[i]));
            return HB_EINVAL;
        }
    }
    const int n = p->n;
    parallel_for(count, count >= 64 ? 0 : 1, [&](size_t idx) {
        Stream r(seed, (DOM_ENC << 56) | ((stream & 0xFFFFFull) << 32) | (first_index + (uint64_t)idx));
        uint32_t *ct = out + idx * out_stride;
        for (int a = 0; a < n; a++) ct[a] = r.u32();
        const uint32_t mu = bits[idx] ? (1u << 29) : (0u - (1u << 29));
        ct[n] = lwe_dot(ct, lwe_key, n) + r.gauss_torus(p->lwe_stdev) + mu;
        for (size_t w = (size_t)n + 1; w < out_stride; w++) ct[w] = 0;
    });
    return HB_OK;
}

int hb_phase(const hb_params *p, const uint32_t *lwe_key, const uint32_t *cts, size_t count,
             size_t stride, int32_t *phase_out) {
    if (!params_ok(p) || stride < (size_t)p->n + 1 || (count && (!cts || !phase_out))) {
        set_error("hb_phase: bad arguments");
        return HB_EINVAL;
    }
    for (size_t i = 0; i < count; i++) {
        const uint32_t *ct = cts + i * stride;
        phase_out[i] = (int32_t)(ct[p->n] - lwe_dot(ct, lwe_key, p->n));
    }
    return HB_OK;
}

int hb_decrypt(const hb_params *p, const uint32_t *lwe_key, const uint32_t *cts, size_t count,
               size_t stride, uint8_t *bits_out) {
    if (!params_ok(p) || stride < (size_t)p->n + 1 || (count && (!cts || !bits_out))) {
        set_error("hb_decrypt: bad arguments");
        return HB_EINVAL;
    }
    for (size_t i = 0; i < count; i++) {
        const uint32_t *ct = cts + i * stride;
        bits_out[i] = (int32_t)(ct[p->n] - lwe_dot(ct, lwe_key, p->n)) > 0 ? 1 : 0;
    }
    return HB_OK;
}

}  // extern "C"
