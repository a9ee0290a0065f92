// reach.cu — Alg. 1 precompute_reachability on the device for slot geometries beyond the loaded tables
// ("on-device reachability precompute for larger state spaces").
//
// The library's geometries have at most 8 memory slots, so mig_geometry_load enumerates Alg. 1 on the host over
// <= 256 occupancy masks. This entry point computes the same table for up to 24 slots (2^24 masks) on the GPU.
// A partition state is a set of disjoint placements; its reachable final states are the states
// obtained by adding placements in its free slots until none fits (R2), so they depend only on its occupancy m
// (R3). With D[t] = the number of distinct placement sets whose union is exactly t:
//   states with occupancy m   D[m]              (|S| = sum of D)
//   final occupancies         D[m] > 0 and no placement fits in the free slots of m  (|F| = sum of D over them)
//   fcr[m]                    sum over t within the free slots of m with m | t final of D[t]
// D by popcount level: the lowest occupied slot of t lies in exactly one placement of each decomposition, and
// that placement starts there, so D[t] = sum over placements q starting at the lowest slot of t, q within t, of
// D[t \ q] (D[0] = 1). fcr enumerates the submasks of each state's free slots (3^n submask visits in total): one
// thread per state with few free slots, one CTA per state with many (split by its highest free slots).
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "device_common.cuh"

namespace mig {

constexpr uint32_t kReachMaxSlots = 24, kReachMaxPlacements = 1024;
constexpr uint32_t kHeavyFree = 12;  // states with more free slots get a CTA each
constexpr uint32_t kSplitBits = 8;   // a heavy state's 2^8 highest-free-slot assignments, one per thread
constexpr uint32_t kCountMax = 0xFFFFFFFFu;

struct ReachParams {
    uint32_t n_slots, n_pl;
    const uint32_t* grp_off;  // placements by lowest slot: masks[grp_off[i] .. grp_off[i+1])
    const uint32_t* masks;
    uint32_t* D;              // decompositions of each occupancy (0 = not a state)
    uint8_t* flags;           // bit 0 = state, bit 1 = final
    uint32_t* fcr;
    uint32_t* heavy;          // states with > kHeavyFree free slots
    unsigned long long* stats;  // [0] states (sum D), [1] finals (sum D), [2] heavy count, [3] overflow
};

// Level k: every occupancy with k occupied slots.
__global__ void k_reach_states(const ReachParams P, uint32_t k) {
    const uint32_t N = 1u << P.n_slots;
    for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x; m < N; m += gridDim.x * blockDim.x) {
        if ((uint32_t)__popc(m) != k) continue;
        uint64_t d = 0;
        if (k == 0) {
            d = 1;  // s0: the unpartitioned GPU
        } else {
            const uint32_t lb = (uint32_t)__ffs(m) - 1u;
            for (uint32_t i = __ldg(P.grp_off + lb), e = __ldg(P.grp_off + lb + 1); i < e; ++i) {
                const uint32_t q = __ldg(P.masks + i);
                if ((q & ~m) == 0) d += P.D[m ^ q];
            }
        }
        if (d > kCountMax) {
            atomicOr(P.stats + 3, 1ull);
            d = kCountMax;
        }
        P.D[m] = (uint32_t)d;
    }
}

__global__ void k_reach_finals(const ReachParams P) {
    const uint32_t N = 1u << P.n_slots;
    unsigned long long ns = 0, nf = 0;
    for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x; m < N; m += gridDim.x * blockDim.x) {
        const uint32_t d = P.D[m];
        uint8_t f = 0;
        if (d) {
            ns += d;
            bool fits = false;
            for (uint32_t i = 0; i < P.n_pl && !fits; ++i) fits = (__ldg(P.masks + i) & m) == 0;
            f = fits ? 1 : 3;
            if (!fits) nf += d;
        }
        P.flags[m] = f;
    }
    for (int o = 16; o > 0; o >>= 1) {
        ns += __shfl_down_sync(FULL, ns, o);
        nf += __shfl_down_sync(FULL, nf, o);
    }
    if ((threadIdx.x & 31u) == 0) {
        if (ns) atomicAdd(P.stats + 0, ns);
        if (nf) atomicAdd(P.stats + 1, nf);
    }
}

__device__ __forceinline__ void store_fcr(const ReachParams& P, uint32_t m, uint64_t c) {
    if (c > kCountMax) {
        atomicOr(P.stats + 3, 1ull);
        c = kCountMax;
    }
    P.fcr[m] = (uint32_t)c;
}

// fcr of the states with few free slots (one thread each); the others are queued for k_reach_fcr_heavy.
__global__ void k_reach_fcr_light(const ReachParams P) {
    const uint32_t N = 1u << P.n_slots, full = N - 1u;
    for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x; m < N; m += gridDim.x * blockDim.x) {
        if (!(P.flags[m] & 1u)) {
            P.fcr[m] = 0;
            continue;
        }
        const uint32_t free = full & ~m;
        if ((uint32_t)__popc(free) > kHeavyFree) {
            const unsigned long long k = atomicAdd(P.stats + 2, 1ull);
            P.heavy[k] = m;
            continue;
        }
        uint64_t c = 0;
        uint32_t s = free;
        for (;;) {  // every submask s of the free slots, free down to 0
            if (P.flags[m | s] & 2u) c += P.D[s];
            if (!s) break;
            s = (s - 1u) & free;
        }
        store_fcr(P, m, c);
    }
}

// One CTA per heavy state: thread t fixes the state's kSplitBits highest free slots to the bits of t and enumerates
// the submasks of the remaining free slots.
__global__ void k_reach_fcr_heavy(const ReachParams P) {
    const uint32_t full = (1u << P.n_slots) - 1u;
    const unsigned long long nh = P.stats[2];
    __shared__ unsigned long long red[32];
    for (unsigned long long h = blockIdx.x; h < nh; h += gridDim.x) {
        const uint32_t m = P.heavy[h];
        uint32_t lo = full & ~m, hs = 0;
        for (uint32_t b = 0; b < kSplitBits; ++b) {  // the kSplitBits highest free slots, deposited from t
            const uint32_t top = 31u - __clz(lo);
            lo &= ~(1u << top);
            if ((threadIdx.x >> (kSplitBits - 1u - b)) & 1u) hs |= 1u << top;
        }
        unsigned long long c = 0;
        uint32_t s = lo;
        for (;;) {
            const uint32_t x = s | hs;
            if (P.flags[m | x] & 2u) c += P.D[x];
            if (!s) break;
            s = (s - 1u) & lo;
        }
        for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(FULL, c, o);
        if ((threadIdx.x & 31u) == 0) red[threadIdx.x >> 5] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long tot = 0;
            for (uint32_t w = 0; w < blockDim.x / 32; ++w) tot += red[w];
            store_fcr(P, m, tot);
        }
        __syncthreads();
    }
}

}  // namespace mig

extern "C" mig_status mig_reachability(uint32_t n_slots, const uint32_t* placement_masks, uint32_t n_placements,
                                       uint32_t* fcr, uint8_t* state_flags, mig_reach_info* info, void* stream) {
    using namespace mig;
    mig_set_launches(0);
    if (n_slots < 1 || n_slots > kReachMaxSlots)
        return mig_set_error(MIG_E_INVALID_ARG, "mig_reachability: n_slots must be 1..24");
    if (!placement_masks || n_placements < 1 || n_placements > kReachMaxPlacements)
        return mig_set_error(MIG_E_INVALID_ARG, "mig_reachability: 1..1024 placements required");
    if (!fcr || !info) return mig_set_error(MIG_E_INVALID_ARG, "mig_reachability: fcr and info are required");
    const uint32_t full = (uint32_t)((1ull << n_slots) - 1ull);
    // placements grouped by their lowest slot (CSR)
    std::vector<uint32_t> off(n_slots + 1, 0), masks;
    for (uint32_t i = 0; i < n_placements; ++i) {
        const uint32_t q = placement_masks[i];
        if (q == 0 || (q & ~full))
            return mig_set_error(MIG_E_INVALID_ARG, "mig_reachability: placement " + std::to_string(i) +
                                                        " is empty or outside the slots");
        ++off[__builtin_ctz(q) + 1];
    }
    for (uint32_t i = 0; i < n_slots; ++i) off[i + 1] += off[i];
    masks.resize(n_placements);
    {
        std::vector<uint32_t> pos(off.begin(), off.end() - 1);
        for (uint32_t i = 0; i < n_placements; ++i) masks[pos[__builtin_ctz(placement_masks[i])]++] = placement_masks[i];
    }
    cudaStream_t s = (cudaStream_t)stream;
    const size_t N = (size_t)1 << n_slots;
    const size_t a = 256;
    auto al = [&](size_t x) { return (x + a - 1) / a * a; };
    const size_t b_off = al((n_slots + 1) * 4), b_masks = al(n_placements * 4), b_stats = al(4 * 8),
                 b_flags = state_flags ? 0 : al(N), b_heavy = al(N * 4), b_D = al(N * 4);
    uint8_t* scr = nullptr;
    cudaError_t e = mig_scratch_alloc((void**)&scr, b_off + b_masks + b_stats + b_flags + b_heavy + b_D, s);
    if (e != cudaSuccess) return mig_set_error(MIG_E_CUDA, std::string("mig_reachability scratch: ") + cudaGetErrorString(e));
    ReachParams P;
    P.n_slots = n_slots;
    P.n_pl = n_placements;
    P.grp_off = reinterpret_cast<uint32_t*>(scr);
    P.masks = reinterpret_cast<uint32_t*>(scr + b_off);
    P.stats = reinterpret_cast<unsigned long long*>(scr + b_off + b_masks);
    P.flags = state_flags ? state_flags : scr + b_off + b_masks + b_stats;
    P.heavy = reinterpret_cast<uint32_t*>(scr + b_off + b_masks + b_stats + b_flags);
    P.D = reinterpret_cast<uint32_t*>(scr + b_off + b_masks + b_stats + b_flags + b_heavy);
    P.fcr = fcr;
    unsigned long long st[4] = {0, 0, 0, 0};
    e = cudaMemcpyAsync((void*)P.grp_off, off.data(), (n_slots + 1) * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync((void*)P.masks, masks.data(), n_placements * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(P.stats, 0, 4 * 8, s);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)std::min<size_t>((size_t)sms * 8, (N + 255) / 256);
    uint32_t launches = 0;
    for (uint32_t k = 0; k <= n_slots && e == cudaSuccess; ++k) {
        k_reach_states<<<grid, 256, 0, s>>>(P, k);
        e = cudaGetLastError();
        ++launches;
    }
    if (e == cudaSuccess) {
        k_reach_finals<<<grid, 256, 0, s>>>(P);
        e = cudaGetLastError();
        ++launches;
    }
    if (e == cudaSuccess) {
        k_reach_fcr_light<<<grid, 256, 0, s>>>(P);
        e = cudaGetLastError();
        ++launches;
    }
    if (e == cudaSuccess && n_slots > kHeavyFree) {
        k_reach_fcr_heavy<<<(unsigned)sms * 4, 1u << kSplitBits, 0, s>>>(P);
        e = cudaGetLastError();
        ++launches;
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(st, P.stats, sizeof(st), cudaMemcpyDeviceToHost, s);
    uint32_t f0 = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&f0, fcr, 4, cudaMemcpyDeviceToHost, s);
    mig_scratch_free(scr, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return mig_set_error(MIG_E_CUDA, std::string("mig_reachability: ") + cudaGetErrorString(e));
    if (st[3]) return mig_set_error(MIG_E_CAPACITY, "mig_reachability: a state or fcr count exceeds 2^32 - 1");
    info->n_states = st[0];
    info->n_finals = st[1];
    info->fcr_s0 = f0;
    mig_set_launches(launches);
    return MIG_OK;
}
