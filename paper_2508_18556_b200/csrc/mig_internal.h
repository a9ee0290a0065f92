// mig_internal.h — internal structures of libmig.so (not part of the C ABI).
#pragma once

#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include "mig.h"

namespace mig {

constexpr int kMaxSlots = MIG_MAX_SLOTS;
constexpr int kMaxProf = MIG_MAX_PROFILES;
constexpr int kMaxLevels = MIG_MAX_LEVELS;
constexpr int kMaxPlace = 8;  // starts per profile (<= slots)

// Geometry parameter block passed BY VALUE to every kernel (lives in the constant bank; uniform-index reads are
// free, lane-divergent tables are copied to shared memory by the kernel prologue).
struct DevGeom {
    uint32_t n_slots, slot_mib, n_compute, n_prof, n_levels, full_prof, full_mem;
    uint32_t n_layout;
    uint32_t mem[16];        // profile memory MiB
    uint32_t comp[16];       // profile compute slices
    uint32_t lenmask[16];    // (1 << memory_slots) - 1
    uint32_t level[16];      // index of mem[p] among the distinct memory levels
    uint32_t wave_cap[16];   // sms_per_slice * comp * warps_per_sm (warp folding, R30)
    uint32_t n_place[16];    // legal starts per profile
    uint32_t place[16][8];   // start | (mask << 8)
    uint32_t level_mem[8];   // distinct memories, ascending
    uint32_t level_next[8];  // next larger memory after level l (0 = none, R14)
    uint32_t layout_prof[8], layout_start[8];
    uint32_t pinfo[16];      // packed: level | comp << 4 | lenmask << 8 | len << 16 | prof << 20
    uint32_t n_alay[8];      // Scheme A: slices of the homogeneous layout of memory level l (0 = none)
    uint32_t alay[8][8];     // start | prof << 8, ascending start
    uint16_t fcr[256];       // fcr by occupancy mask (0 = not a valid occupancy)
};

}  // namespace mig

struct mig_geometry {
    std::string name;
    mig_geometry_info info;
    std::vector<std::string> prof_names;
    mig::DevGeom dg;
    uint32_t sms_per_slice = 0, warps_per_sm = 0;
    // Slot-level partition states (occupancy, instance starts) reachable by placements, and for every state and
    // placement q (index = sum of earlier profiles' starts + k): {fcr(result) << 16 | (15 - #destroyed) << 8 |
    // start, destroyed-slot mask | next state << 8}, where placing q destroys the instances it overlaps (Alg. 2
    // when nothing overlaps; fusion / fission R8 otherwise). Used by the lane kernel's FUSION_FISSION path.
    std::vector<uint32_t> trans;       // [n_trans_states][n_q][2]
    std::vector<int32_t> trans_id;     // state id by occ | start mask << 8 (-1 = not a reachable state)
    std::vector<uint16_t> sid16;       // the same as u16 (0xFFFF = unreachable): the device copy the lane kernel reads
    uint32_t n_trans_states = 0, n_q = 0;
    // Fusion / fission answers (R8) by (state, profile p, candidate mask c over p's placements): the entry of the
    // best placement k in c that overlaps an instance ({0, 0} if none). Row = n_a7 entries, profile p's block
    // starts at sum over earlier profiles of 2^n_place.
    std::vector<uint32_t> a7;          // [n_trans_states][n_a7][2]
    uint32_t n_a7 = 0;
    std::mutex mu;                     // guards dev[], sid_dev[], a7_dev[]
    mig::DevGeom* dev[64] = {};        // per-device copy, uploaded on first use
    uint16_t* sid_dev[64] = {};
    uint32_t* a7_dev[64] = {};
    ~mig_geometry();
};

// Stream-ordered library scratch from a private memory pool per device (capi.cu): allocations persist in the pool
// between calls (no re-mapping of large scratch every call) without changing the device's default pool, which
// other users of the process share; mig_release_scratch() trims it.
#include <cuda_runtime.h>
cudaError_t mig_scratch_alloc(void** p, size_t bytes, cudaStream_t s);
cudaError_t mig_scratch_free(void* p, cudaStream_t s);

// error helpers (capi.cu)
mig_status mig_set_error(mig_status s, const std::string& msg);
void mig_note_launches(uint32_t n);
void mig_set_launches(uint32_t n);

// mig_timing_enable support (capi.cu): when timing is on for this thread, records events on `stream` around the
// launches issued by f (f returns a cudaError_t and the number of launches through its argument) under `name`.
#include <functional>
typedef struct CUstream_st* mig_stream_t;
int mig_timed(const char* name, mig_stream_t stream, const std::function<int(uint32_t*)>& f);
