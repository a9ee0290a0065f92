// simulate_sa.cu — k_sa_group: Scheme A's grouping pass (R38, PAPER.md Scheme A) as its own launch ahead of the
// lane kernel (simulate_lane.cu reads its grouped records sequentially). MIG_SA_PREGROUP=0 keeps the grouping inside
// the lane kernel instead (A/B and parity of both paths).
#include <algorithm>

#include "lane_common.cuh"

namespace mig {

// ================================================================================================================
// k_sa_group: Scheme A's grouping pass (sorted_by_mig_group, reading R38) as its own launch before
// the Scheme A lane launch. One warp per trace (four per CTA): its job records 32 at a time (coalesced), the tight
// fits in parallel, group positions by ballots (no event loop); the t = 0 REJECT records (queue order) go into the trace's decision
// hash, and the records are written in group order (ascending memory level of the tight fit, queue order within a
// level) with their x word replaced by the job index (and, without a dext buffer, the workspace added to the true
// footprint: only warp folding / wave time need the rest of the extension record), so the lane kernel dispatches each group by reading the next
// record of the group sequentially instead of re-reading records by job index. Per trace: sa_hdr[2t]
// = {len0 | len1 << 16, len2 | len3 << 16, len4 | rejected << 16, error bits}, sa_hdr[2t + 1] = {hash lo, hash hi}.
// Pass 1 counts the groups (and the REJECT hash), pass 2 scatters (the trace's records are re-read from L2).
// ================================================================================================================
template <bool XR>
__global__ void __launch_bounds__(kLaneThreads) k_sa_group(const DevGeom* __restrict__ Gg, const LaneParams P,
                                                          uint4* desc, uint4* dext, uint4* hdr) {
    __shared__ uint32_t s_lmem[8];
    __shared__ uint8_t s_first[8];
    __shared__ DevGeom sG;
    const uint32_t tid = threadIdx.x, lane = tid & 31u;
    {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(Gg);
        uint32_t* dst = reinterpret_cast<uint32_t*>(&sG);
        for (uint32_t i = tid; i < sizeof(DevGeom) / 4; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    const DevGeom& G = sG;
    if (tid < 8) {
        uint32_t f = 0xFFu;
        for (uint32_t p = G.n_prof; p-- > 0;)
            if (G.level[p] == tid) f = p;
        s_first[tid] = (uint8_t)(tid < G.n_levels ? f : 0xFFu);
        s_lmem[tid] = tid < G.n_levels ? G.level_mem[tid] : 0xFFFFFFFFu;
    }
    __syncthreads();
    const bool fold = (P.pol.flags & MIG_WARP_FOLD) != 0;
    // the tight fit of lane_tight_fit<MIG_SCHEME_A> (R6, R30)
    auto fit = [&](uint32_t req, uint32_t warps) -> uint32_t {
        if (!fold || warps == 0) {
            uint32_t L = s_lmem[3] < req ? 4u : 0u;
            L += s_lmem[L + 1] < req ? 2u : 0u;
            L += s_lmem[L] < req ? 1u : 0u;
            return s_first[L];
        }
        const uint32_t cf = G.wave_cap[G.full_prof];
        for (uint32_t p = 0; p < G.n_prof; ++p) {
            if (G.mem[p] < req) continue;
            const uint32_t cp = G.wave_cap[p];
            if ((warps + cp - 1) / cp != (warps + cf - 1) / cf) continue;
            return p;
        }
        return kNoNeed;
    };
    const uint64_t jbase = P.off[0];
    const uint32_t ctx = P.ctx, mem0 = G.mem[0];
    const uint32_t lt = (1u << lane) - 1u;  // lanes below this one
    // one warp per trace: its records 32 at a time (coalesced), the tight fits in parallel, the group positions by
    // ballots; the REJECT records (rare) folded into the hash in queue order by lane 0
    for (unsigned long long tr = blockIdx.x * (kLaneThreads / 32) + (tid >> 5); tr < P.n_traces;
         tr += (unsigned long long)gridDim.x * (kLaneThreads / 32)) {
        const uint64_t o0 = P.off[tr], o1 = P.off[tr + 1], j0 = o0 - jbase;
        uint32_t n = (uint32_t)(o1 - o0), err = 0;
        if (o1 - o0 > P.max_jobs) {
            err = (uint32_t)MIG_ERR_TRACE_TOO_LONG;
            n = 0;
        }
        uint32_t hl = (uint32_t)kFnvOffset, hh = (uint32_t)(kFnvOffset >> 32), rej = 0;
        uint32_t cnt[5] = {0, 0, 0, 0, 0};
        auto need_of = [&](uint32_t k, uint4& r, uint4& e) -> uint32_t {
            r = __ldg(P.jobs + j0 + k);
            e = XR ? __ldg(P.ext + j0 + k) : make_uint4(0, 0, 0, 0);
            const uint32_t cls = (r.z >> 16) & 0xFFu;
            return fit(cls == kClassDynamic ? mem0 : r.x + e.x + ctx, e.y);  // R16 / est + ws + ctx
        };
        for (uint32_t c = 0; c < n; c += 32) {  // pass 1: REJECTs in queue order, group sizes
            const uint32_t k = c + lane;
            uint32_t lv = 0xFFu;
            bool rj = false;
            if (k < n) {
                uint4 r, e;
                const uint32_t need = need_of(k, r, e);
                const uint32_t cls = (r.z >> 16) & 0xFFu, T = r.z & 0xFFFFu;
                if (cls > 2 || T > 4096) err |= (uint32_t)MIG_ERR_BAD_RECORD;
                rj = need == kNoNeed;
                if (!rj) lv = G.level[need];
            }
            uint32_t rm = __ballot_sync(FULL, rj);
            rej += __popc(rm);
            while (rm) {  // lane-uniform loop over this chunk's REJECTs, in queue order
                const uint32_t q = (uint32_t)__ffs(rm) - 1u;
                rm &= rm - 1u;
                lrec(hl, hh, 0u, ((c + q) << 16) | (K_REJECT << 12) | 0xFF0u);
            }
#pragma unroll
            for (int l = 0; l < 5; ++l) cnt[l] += __popc(__ballot_sync(FULL, lv == (uint32_t)l));
        }
        uint32_t pos[5];
        pos[0] = 0;
#pragma unroll
        for (int l = 1; l < 5; ++l) pos[l] = pos[l - 1] + cnt[l - 1];
        for (uint32_t c = 0; c < n; c += 32) {  // pass 2: the records in group order, x = the job index
            const uint32_t k = c + lane;
            uint4 r = make_uint4(0, 0, 0, 0), e = r;
            uint32_t lv = 0xFFu;
            if (k < n) {
                const uint32_t need = need_of(k, r, e);
                if (need != kNoNeed) lv = G.level[need];
            }
            uint32_t at = 0;
#pragma unroll
            for (int l = 0; l < 5; ++l) {
                const uint32_t m = __ballot_sync(FULL, lv == (uint32_t)l);
                if (lv == (uint32_t)l) at = pos[l] + __popc(m & lt);
                pos[l] += __popc(m);
            }
            if (lv != 0xFFu) {
                r.x = k;
                if (XR && !dext && ((r.z >> 16) & 0xFFu) != kClassDynamic)  // true + ws (saturating, as the lane
                    r.y = r.y + e.x < r.y ? 0xFFFFFFFFu : r.y + e.x;          // kernel's 64-bit sum): no dext needed
                desc[j0 + at] = r;
                if (XR && dext) dext[j0 + at] = e;
            }
        }
        err = __reduce_or_sync(FULL, err);
        if (lane == 0) {
            hdr[2 * tr] = make_uint4(cnt[0] | (cnt[1] << 16), cnt[2] | (cnt[3] << 16), cnt[4] | (rej << 16), err);
            hdr[2 * tr + 1] = make_uint4(hl, hh, 0u, 0u);
        }
    }
}


cudaError_t launch_sa_group(const DevGeom* Gdev, const LaneParams& P, uint4* desc, uint4* dext, uint4* hdr,
                            int sm_count, cudaStream_t stream) {
    // a warp per trace, four traces per CTA
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)sm_count * 16,
                                                                             (P.n_traces + 3) / 4));
    if (P.ext) k_sa_group<true><<<grid, kLaneThreads, 0, stream>>>(Gdev, P, desc, dext, hdr);
    else k_sa_group<false><<<grid, kLaneThreads, 0, stream>>>(Gdev, P, desc, nullptr, hdr);
    return cudaGetLastError();
}

}  // namespace mig
