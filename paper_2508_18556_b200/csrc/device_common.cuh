// device_common.cuh — device-side helpers shared by the estimation and simulation kernels of libmig.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "mig_internal.h"

namespace mig {

constexpr uint32_t FULL = 0xFFFFFFFFu;
constexpr uint32_t kNever = MIG_NEVER;
constexpr uint32_t kClassDynamic = 2;
constexpr int kMaxPolicies = 8;

// Decision-record kinds: the per-trace FNV-1a-64 hash covers every decision and
// applied event in order, so oracle/GPU parity of the hash is parity of every placement and event time.
enum : uint32_t {
    K_REUSE = 1, K_ALLOC = 2, K_RECONF = 3, K_WAIT = 4, K_REJECT = 5, K_COMPLETE = 6, K_OOM = 7, K_PREEMPT = 8,
    K_FAILED = 9, K_PLACE_STATIC = 10, K_PLACE_BASELINE = 11, K_LAYOUT = 12, K_PLACE_GROUP = 13
};

constexpr uint64_t kFnvOffset = 0xcbf29ce484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001b3ull;

__device__ __forceinline__ void hash_record(uint64_t& h, uint32_t tick, uint32_t job, uint32_t kind, uint32_t start,
                                            uint32_t prof, uint32_t nd) {
    uint32_t lo = ((job & 0xFFFFu) << 16) | ((kind & 0xFu) << 12) | ((start & 0xFu) << 8) | ((prof & 0xFu) << 4) |
                  (nd & 0xFu);
    uint64_t r = ((uint64_t)tick << 32) | lo;
    h = (h ^ r) * kFnvPrime;
}

// Canonical int128 -> double: sign-magnitude, hi*2^64 + lo, each u64
// conversion and the addition rounded to nearest. Identical sequence to the oracle's.
__device__ __forceinline__ double i128_to_double(__int128 x) {
    const int64_t lo64 = (int64_t)x;
    if ((__int128)lo64 == x) return __ll2double_rn(lo64);  // same single rounding as the canonical form
    bool neg = x < 0;
    unsigned __int128 m = neg ? (unsigned __int128)(-x) : (unsigned __int128)x;
    uint64_t hi = (uint64_t)(m >> 64), lo = (uint64_t)m;
    double d = __dadd_rn(__dmul_rn(__ull2double_rn(hi), 18446744073709551616.0), __ull2double_rn(lo));
    return neg ? -d : d;
}

// Warp inclusive prefix sum of a 64-bit value.
__device__ __forceinline__ int64_t warp_scan_i64(int64_t v, uint32_t lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int64_t o = __shfl_up_sync(FULL, v, d);
        if (lane >= (uint32_t)d) v += o;
    }
    return v;
}

}  // namespace mig
