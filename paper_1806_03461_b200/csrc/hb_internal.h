// Internal declarations shared by the host (hb_host.cpp) and device
// (hb_engine.cu) halves of libhebnn_b200.so.
#pragma once

#include <cstdint>
#include <string>

#include "../../include/hebnn_b200.h"

namespace hb {

// The kernels are specialised for BASELINE.json configs[0]: N = 1024, k = 1,
// Bg = 2^7, l = 3, KS base 2^2, t = 8.  n (LWE dimension) is a runtime value.
constexpr int kN = 1024;          // ring degree
constexpr int kNH = 512;          // complex FFT length (negacyclic fold)
constexpr int kL = 3;             // gadget length
constexpr int kBgBits = 7;        // log2 Bg
constexpr int kRows = 2 * kL;     // TGSW rows, (k+1) l
constexpr int kKsBaseBits = 2;
constexpr int kKsT = 8;
constexpr int kKsVals = (1 << kKsBaseBits) - 1;  // non-zero digit values
constexpr int kMaxLweN = 1023;
constexpr int kBigStride = 1028;  // words per extracted LWE (kN + 1, padded to 16 B)
constexpr int kKskStride = 640;   // words per device KSK row (n + 1 padded)
constexpr int kMaxKsN = kKskStride - 1;  // largest n the key switch covers (n + 1 output columns)
static_assert(kMaxKsN <= kMaxLweN, "key-switch columns exceed the mod-switch buffers");

void set_error(const std::string &msg);
bool params_ok(const hb_params *p);
int bk_unroll(const hb_params *p);          // 1 or 2 (0 reads as 1)
size_t bk_tgsw_count(const hb_params *p);   // TGSW samples in the bootstrapping key

// Bootstrapped-gate work items produced from hb_gate records.
constexpr uint32_t kNoItem = 0xFFFFFFFFu;
constexpr uint32_t kKsSub = 0x80000000u;  // KsItem::i1 flag: subtract big[i1] instead of adding it
struct BrItem {      // lin = (0, c0) + alpha * pool[src_a] + beta * pool[src_b] + gamma * pool[src_c]
    uint32_t src_a, src_b, src_c, c0;
    int32_t coef;    // alpha in bits 0..7, beta in bits 8..15, gamma in bits 16..23 (signed bytes)
    uint32_t x2;     // kNoItem, or the big-LWE row (item units) of a second extraction at index N/2 (HA)
};
struct KsItem {      // pool[dst] = KS(big[i0] (+/- big[i1 & ~kKsSub]) + (0, cadd)); i1 = kNoItem: big[i0] only
    uint32_t dst, i0, i1, cadd;
};

}  // namespace hb
