// geometry.cpp — mig_geometry_load and the host-side tables of the partition manager.
//
// The partition state machine M = (S, Sigma, delta, s0, F) of PAPER.md:496-514 is represented on the device by
// the OCCUPANCY BITMASK of the memory slots (bit i = slot i belongs to an instance). Alg. 1 is
// precomputed here once per geometry as fcr[occ]: the number of distinct fully configured states (maximal sets of
// placed instances, reading R2/R3) that extend a state with occupancy occ. The count depends only on occ because
// a state's extensions are exactly the maximal tilings of its free slots; this requires that the compute-slice
// limit never binds, which load() checks. The enumeration below walks slots left to right and either leaves a
// slot empty for good or starts one placement there, so every instance set is produced exactly once.
#include <dlfcn.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <fstream>
#include <sstream>

#include "json_min.h"
#include "mig_internal.h"

namespace {

using mig::DevGeom;

struct Pl {
    uint32_t prof, start, mask;
};

struct Tables {
    uint32_t n_slots, n_compute;
    std::vector<Pl> pl;
    std::vector<uint32_t> comp;
};

// Maximal tilings of the free slots of `free_left` from slot s on. empty_set = slots decided to stay empty.
// If comp_max != nullptr, records the largest total compute of any completed maximal set (base_comp included).
uint64_t count_maximal(const Tables& T, uint32_t s, uint32_t free_left, uint32_t empty_set, uint32_t base_comp,
                       uint32_t* comp_max) {
    while (s < T.n_slots && !((free_left >> s) & 1u)) ++s;
    if (s >= T.n_slots) {
        for (const Pl& p : T.pl)
            if ((p.mask & ~empty_set) == 0) return 0;  // some placement still fits: not fully configured
        if (comp_max && base_comp > *comp_max) *comp_max = base_comp;
        return 1;
    }
    uint64_t n = count_maximal(T, s + 1, free_left & ~(1u << s), empty_set | (1u << s), base_comp, comp_max);
    for (const Pl& p : T.pl)
        if (p.start == s && (p.mask & ~free_left) == 0)
            n += count_maximal(T, s + 1, free_left & ~p.mask, empty_set, base_comp + T.comp[p.prof], comp_max);
    return n;
}

// Slot-level transition table (mig_geometry::trans): breadth-first over states (occ, SM) from the empty GPU.
// Placing q = (profile, start) destroys the instances whose slots it overlaps (the instances are the runs of
// occupied slots cut at instance starts) and creates q. Left empty (n_q = 0) if the table would not fit 24-bit
// state ids or 64 placements.
void build_transitions(mig_geometry* g) {
    const DevGeom& d = g->dg;
    std::vector<uint32_t> qs;  // start | mask << 8, in (profile, k) order
    for (uint32_t p = 0; p < d.n_prof; ++p)
        for (uint32_t k = 0; k < d.n_place[p]; ++k) qs.push_back(d.place[p][k]);
    g->trans.clear();
    g->a7.clear();
    g->n_q = g->n_a7 = g->n_trans_states = 0;
    if (qs.size() > 64) return;
    const uint32_t nq = (uint32_t)qs.size();
    std::vector<uint32_t> keys{0};  // occ | SM << 8
    std::vector<int32_t> id(1u << 16, -1);
    id[0] = 0;
    std::vector<uint32_t> tab;
    for (size_t i = 0; i < keys.size(); ++i) {
        const uint32_t occ = keys[i] & 0xFFu, SM = keys[i] >> 8;
        uint32_t EM = 0;  // last slot of every instance
        for (uint32_t s = 0; s < d.n_slots; ++s) {
            if (!((SM >> s) & 1u)) continue;
            uint32_t e = s;
            while (e + 1 < d.n_slots && ((occ >> (e + 1)) & 1u) && !((SM >> (e + 1)) & 1u)) ++e;
            EM |= 1u << e;
        }
        for (uint32_t q = 0; q < nq; ++q) {
            const uint32_t lo = qs[q] & 0xFFu, qm = qs[q] >> 8;
            const uint32_t hi = 31u - (uint32_t)__builtin_clz(qm);
            uint32_t a = lo, b = hi;
            if ((occ >> lo) & 1u) a = 31u - (uint32_t)__builtin_clz(SM & ((2u << lo) - 1u));
            if ((occ >> hi) & 1u) b = (uint32_t)__builtin_ctz(EM & ~((1u << hi) - 1u));
            const uint32_t rm = occ & ((2u << b) - 1u) & ~((1u << a) - 1u);
            const uint32_t nocc = (occ & ~rm) | qm, nSM = (SM & ~rm) | (1u << lo);
            const uint32_t nd = (uint32_t)__builtin_popcount(SM & rm);
            const uint32_t key = nocc | (nSM << 8);
            if (id[key] < 0) {
                id[key] = (int32_t)keys.size();
                keys.push_back(key);
            }
            tab.push_back(((uint32_t)d.fcr[nocc] << 16) | ((15u - nd) << 8) | lo);
            tab.push_back(rm | ((uint32_t)id[key] << 8));
        }
        if (keys.size() >= 0xFFFFu) return;  // u16 state ids (the key space is 2^16)
    }
    // fusion / fission answers per (state, profile, candidate mask)
    uint32_t na7 = 0;
    for (uint32_t p = 0; p < d.n_prof; ++p) na7 += 1u << d.n_place[p];
    std::vector<uint32_t> a7((size_t)keys.size() * na7 * 2, 0u);
    for (size_t i = 0; i < keys.size(); ++i) {
        const uint32_t occ = keys[i] & 0xFFu;
        uint32_t base = 0, qb = 0;
        for (uint32_t p = 0; p < d.n_prof; ++p) {
            const uint32_t np = d.n_place[p];
            for (uint32_t c = 0; c < (1u << np); ++c) {
                uint32_t bx = 0, by = 0;
                for (uint32_t k = 0; k < np; ++k) {
                    if (!((c >> k) & 1u) || !((d.place[p][k] >> 8) & occ)) continue;
                    const uint32_t* e = &tab[(i * nq + qb + k) * 2];
                    if (e[0] > bx) {
                        bx = e[0];
                        by = e[1];
                    }
                }
                a7[(i * na7 + base + c) * 2] = bx;
                a7[(i * na7 + base + c) * 2 + 1] = by;
            }
            base += 1u << np;
            qb += np;
        }
    }
    g->sid16.assign(id.size(), 0xFFFFu);
    for (size_t k = 0; k < id.size(); ++k)
        if (id[k] >= 0) g->sid16[k] = (uint16_t)id[k];
    g->trans.swap(tab);
    g->a7.swap(a7);
    g->trans_id.swap(id);
    g->n_q = nq;
    g->n_a7 = na7;
    g->n_trans_states = (uint32_t)keys.size();
}

// All sets of non-overlapping placements inside free_left (|S| when started from the empty GPU).
uint64_t count_all(const Tables& T, uint32_t s, uint32_t free_left) {
    while (s < T.n_slots && !((free_left >> s) & 1u)) ++s;
    if (s >= T.n_slots) return 1;
    uint64_t n = count_all(T, s + 1, free_left & ~(1u << s));
    for (const Pl& p : T.pl)
        if (p.start == s && (p.mask & ~free_left) == 0) n += count_all(T, s + 1, free_left & ~p.mask);
    return n;
}

// Is `occ` exactly a union of non-overlapping placements?
bool tileable(const Tables& T, uint32_t occ) {
    if (occ == 0) return true;
    uint32_t s = (uint32_t)__builtin_ctz(occ);
    for (const Pl& p : T.pl)
        if (p.start == s && (p.mask & ~occ) == 0 && tileable(T, occ & ~p.mask)) return true;
    return false;
}

bool read_file(const std::string& path, std::string* out) {
    std::ifstream f(path, std::ios::binary);
    if (!f) return false;
    std::stringstream ss;
    ss << f.rdbuf();
    *out = ss.str();
    return true;
}

std::string builtin_dir() {
    Dl_info info;
    if (dladdr((void*)&builtin_dir, &info) && info.dli_fname) {
        std::string p = info.dli_fname;
        size_t k = p.find_last_of('/');
        return (k == std::string::npos ? std::string(".") : p.substr(0, k)) + "/geometries/";
    }
    return "geometries/";
}

bool get_u32(const mig::json::Value& o, const char* key, uint32_t* out, std::string* err, bool required = true,
             uint32_t dflt = 0) {
    const mig::json::Value* v = o.get(key);
    if (!v) {
        if (!required) {
            *out = dflt;
            return true;
        }
        *err = std::string("missing field '") + key + "'";
        return false;
    }
    if (v->kind != mig::json::Value::Number || v->num < 0 || v->num > 4294967295.0 || v->num != (double)(uint64_t)v->num) {
        *err = std::string("field '") + key + "' must be a non-negative integer";
        return false;
    }
    *out = (uint32_t)v->num;
    return true;
}

mig_status load_geometry(const std::string& text, mig_geometry* g) {
    mig::json::Value root;
    std::string err;
    mig::json::Parser parser(text);
    if (!parser.parse(&root, &err)) return mig_set_error(MIG_E_PARSE, "geometry JSON: " + err);
    if (root.kind != mig::json::Value::Object) return mig_set_error(MIG_E_PARSE, "geometry JSON: not an object");
    DevGeom& d = g->dg;
    memset(&d, 0, sizeof(d));
    memset(&g->info, 0, sizeof(g->info));
    const mig::json::Value* nm = root.get("gpu_name");
    g->name = nm && nm->kind == mig::json::Value::String ? nm->str : "unnamed";
    uint32_t idle_w, wps;
    if (!get_u32(root, "total_memory_slots", &d.n_slots, &err) || !get_u32(root, "slot_mib", &d.slot_mib, &err) ||
        !get_u32(root, "total_compute_slices", &d.n_compute, &err) ||
        !get_u32(root, "sms_per_slice", &g->sms_per_slice, &err, false, 14) ||
        !get_u32(root, "warps_per_sm", &g->warps_per_sm, &err, false, 64) ||
        !get_u32(root, "idle_w", &idle_w, &err, false, 30) || !get_u32(root, "w_per_slice", &wps, &err, false, 25))
        return mig_set_error(MIG_E_VALIDATION, err);
    if (d.n_slots < 1 || d.n_slots > (uint32_t)mig::kMaxSlots)
        return mig_set_error(MIG_E_VALIDATION, "total_memory_slots must be 1..8");
    if (d.slot_mib == 0 || (uint64_t)d.slot_mib * d.n_slots > 0x7FFFFFFFull)
        return mig_set_error(MIG_E_VALIDATION, "slot_mib out of range");
    if (d.n_compute == 0) return mig_set_error(MIG_E_VALIDATION, "total_compute_slices must be > 0");
    const mig::json::Value* profs = root.get("profiles");
    if (!profs || profs->kind != mig::json::Value::Array || profs->arr.empty())
        return mig_set_error(MIG_E_VALIDATION, "missing or empty 'profiles'");
    if (profs->arr.size() > (size_t)mig::kMaxProf)
        return mig_set_error(MIG_E_VALIDATION, "too many profiles (max 15)");
    Tables T;
    T.n_slots = d.n_slots;
    T.n_compute = d.n_compute;
    d.n_prof = (uint32_t)profs->arr.size();
    g->prof_names.clear();
    for (uint32_t p = 0; p < d.n_prof; ++p) {
        const mig::json::Value& pv = profs->arr[p];
        std::string where = "profiles[" + std::to_string(p) + "]";
        const mig::json::Value* pn = pv.get("name");
        g->prof_names.push_back(pn && pn->kind == mig::json::Value::String ? pn->str : where);
        uint32_t c, len;
        if (!get_u32(pv, "compute_slices", &c, &err) || !get_u32(pv, "memory_slots", &len, &err))
            return mig_set_error(MIG_E_VALIDATION, where + ": " + err);
        if (c == 0 || c > d.n_compute) return mig_set_error(MIG_E_VALIDATION, where + ".compute_slices out of range");
        if (len == 0 || len > d.n_slots) return mig_set_error(MIG_E_VALIDATION, where + ".memory_slots out of range");
        const mig::json::Value* st = pv.get("starts");
        if (!st || st->kind != mig::json::Value::Array || st->arr.empty() || st->arr.size() > (size_t)mig::kMaxPlace)
            return mig_set_error(MIG_E_VALIDATION, where + ".starts must list 1..8 slots");
        d.mem[p] = len * d.slot_mib;
        d.comp[p] = c;
        d.lenmask[p] = (1u << len) - 1u;
        d.wave_cap[p] = g->sms_per_slice * c * g->warps_per_sm;
        d.n_place[p] = 0;
        uint32_t prev = 0;
        for (size_t k = 0; k < st->arr.size(); ++k) {
            const mig::json::Value& sv = st->arr[k];
            if (sv.kind != mig::json::Value::Number || sv.num < 0 || sv.num != (double)(int)sv.num)
                return mig_set_error(MIG_E_VALIDATION, where + ".starts[" + std::to_string(k) + "] not an integer");
            uint32_t s = (uint32_t)sv.num;
            if (s + len > d.n_slots)
                return mig_set_error(MIG_E_VALIDATION, where + ".starts[" + std::to_string(k) +
                                                           "]: placement exceeds the memory slots");
            if (k > 0 && s <= prev)
                return mig_set_error(MIG_E_VALIDATION, where + ".starts must be strictly increasing");
            prev = s;
            uint32_t mask = d.lenmask[p] << s;
            d.place[p][d.n_place[p]++] = s | (mask << 8);
            T.pl.push_back({p, s, mask});
        }
        T.comp.push_back(c);
        if (p > 0 && (d.mem[p] < d.mem[p - 1] || (d.mem[p] == d.mem[p - 1] && d.comp[p] < d.comp[p - 1])))
            return mig_set_error(MIG_E_VALIDATION, where + ": profiles must be sorted by (memory, compute)");
    }
    d.full_prof = d.n_prof - 1;
    d.full_mem = d.n_slots * d.slot_mib;
    if (d.mem[d.full_prof] != d.full_mem || d.n_place[d.full_prof] != 1 || (d.place[d.full_prof][0] & 0xFF) != 0)
        return mig_set_error(MIG_E_VALIDATION, "the last profile must be the whole GPU (all slots, start 0)");
    // memory levels (distinct profile memories) and the OOM ladder (R14)
    std::vector<uint32_t> L;
    for (uint32_t p = 0; p < d.n_prof; ++p)
        if (L.empty() || L.back() != d.mem[p]) L.push_back(d.mem[p]);
    if (L.size() > (size_t)mig::kMaxLevels)
        return mig_set_error(MIG_E_VALIDATION, "more than 5 distinct profile memory sizes");
    d.n_levels = (uint32_t)L.size();
    for (uint32_t l = 0; l < d.n_levels; ++l) {
        d.level_mem[l] = L[l];
        d.level_next[l] = l + 1 < d.n_levels ? L[l + 1] : 0u;
    }
    for (uint32_t p = 0; p < d.n_prof; ++p) {
        d.level[p] = (uint32_t)(std::find(L.begin(), L.end(), d.mem[p]) - L.begin());
        if (d.comp[p] > 15) return mig_set_error(MIG_E_VALIDATION, "compute_slices above 15 unsupported");
        d.pinfo[p] = d.level[p] | (d.comp[p] << 4) | (d.lenmask[p] << 8) |
                     ((uint32_t)__builtin_popcount(d.lenmask[p]) << 16) | (p << 20);
    }
    // Alg. 1: fcr for every valid occupancy mask
    const uint32_t all = (1u << d.n_slots) - 1u;
    uint32_t comp_max = 0;
    uint64_t n_finals = count_maximal(T, 0, all, 0, 0, &comp_max);
    if (comp_max > d.n_compute)
        return mig_set_error(MIG_E_VALIDATION,
                             "compute slices over-committed by a placement combination (mask-indexed fcr needs "
                             "memory non-overlap to imply compute non-overlap)");
    uint64_t n_states = count_all(T, 0, all);
    if (n_states > 1000000ull) return mig_set_error(MIG_E_CAPACITY, "state space exceeds 1e6 states");
    for (uint32_t occ = 0; occ <= all; ++occ) {
        uint64_t f = tileable(T, occ) ? count_maximal(T, 0, all & ~occ, 0, 0, nullptr) : 0;
        if (f > 0xFFFF) return mig_set_error(MIG_E_CAPACITY, "fcr exceeds 65535");
        d.fcr[occ] = (uint16_t)f;
    }
    // static layout (R11)
    const mig::json::Value* lay = root.get("static_layout");
    uint32_t lay_occ = 0;
    if (lay && lay->kind == mig::json::Value::Array) {
        if (lay->arr.size() > 8) return mig_set_error(MIG_E_VALIDATION, "static_layout: at most 8 instances");
        for (size_t i = 0; i < lay->arr.size(); ++i) {
            const mig::json::Value& e = lay->arr[i];
            std::string where = "static_layout[" + std::to_string(i) + "]";
            if (e.kind != mig::json::Value::Array || e.arr.size() != 2 || e.arr[0].kind != mig::json::Value::String ||
                e.arr[1].kind != mig::json::Value::Number)
                return mig_set_error(MIG_E_VALIDATION, where + " must be [profile_name, start]");
            auto it = std::find(g->prof_names.begin(), g->prof_names.end(), e.arr[0].str);
            if (it == g->prof_names.end()) return mig_set_error(MIG_E_VALIDATION, where + ": unknown profile");
            uint32_t p = (uint32_t)(it - g->prof_names.begin()), s = (uint32_t)e.arr[1].num;
            bool legal = false;
            for (uint32_t k = 0; k < d.n_place[p]; ++k) legal |= (d.place[p][k] & 0xFF) == s;
            uint32_t mask = d.lenmask[p] << s;
            if (!legal || (mask & lay_occ)) return mig_set_error(MIG_E_VALIDATION, where + ": illegal placement");
            lay_occ |= mask;
            d.layout_prof[d.n_layout] = p;
            d.layout_start[d.n_layout] = s;
            d.n_layout++;
        }
    }
    // Scheme A homogeneous layouts, one per memory level (R38; optional)
    const mig::json::Value* al = root.get("scheme_a_layouts");
    if (al && al->kind == mig::json::Value::Array) {
        for (size_t i = 0; i < al->arr.size(); ++i) {
            const mig::json::Value& e = al->arr[i];
            std::string where = "scheme_a_layouts[" + std::to_string(i) + "]";
            uint32_t mm;
            if (!get_u32(e, "memory_mib", &mm, &err)) return mig_set_error(MIG_E_VALIDATION, where + ": " + err);
            auto lit = std::find(L.begin(), L.end(), mm);
            if (lit == L.end()) return mig_set_error(MIG_E_VALIDATION, where + ".memory_mib is not a profile memory");
            const uint32_t lvl = (uint32_t)(lit - L.begin());
            const mig::json::Value* sl = e.get("slices");
            if (!sl || sl->kind != mig::json::Value::Array || sl->arr.empty() || sl->arr.size() > 8)
                return mig_set_error(MIG_E_VALIDATION, where + ".slices must list 1..8 slices");
            uint32_t occ = 0, comp = 0;
            std::vector<std::pair<uint32_t, uint32_t>> v;
            for (size_t k = 0; k < sl->arr.size(); ++k) {
                const mig::json::Value& x = sl->arr[k];
                std::string w2 = where + ".slices[" + std::to_string(k) + "]";
                if (x.kind != mig::json::Value::Array || x.arr.size() != 2 || x.arr[0].kind != mig::json::Value::String ||
                    x.arr[1].kind != mig::json::Value::Number)
                    return mig_set_error(MIG_E_VALIDATION, w2 + " must be [profile_name, start]");
                auto it = std::find(g->prof_names.begin(), g->prof_names.end(), x.arr[0].str);
                if (it == g->prof_names.end()) return mig_set_error(MIG_E_VALIDATION, w2 + ": unknown profile");
                const uint32_t p = (uint32_t)(it - g->prof_names.begin()), st = (uint32_t)x.arr[1].num;
                bool legal = false;
                for (uint32_t q = 0; q < d.n_place[p]; ++q) legal |= (d.place[p][q] & 0xFF) == st;
                const uint32_t mask = d.lenmask[p] << st;
                if (!legal || (mask & occ) || d.mem[p] != mm)
                    return mig_set_error(MIG_E_VALIDATION, w2 + ": illegal or wrong-size slice");
                occ |= mask;
                comp += d.comp[p];
                v.push_back({st, p});
            }
            if (comp > d.n_compute) return mig_set_error(MIG_E_VALIDATION, where + ": compute over-committed");
            std::sort(v.begin(), v.end());
            d.n_alay[lvl] = (uint32_t)v.size();
            for (size_t k = 0; k < v.size(); ++k) d.alay[lvl][k] = v[k].first | (v[k].second << 8);
        }
    }
    build_transitions(g);
    mig_geometry_info& in = g->info;
    snprintf(in.gpu_name, sizeof(in.gpu_name), "%s", g->name.c_str());
    in.n_slots = d.n_slots;
    in.slot_mib = d.slot_mib;
    in.n_compute = d.n_compute;
    in.n_profiles = d.n_prof;
    in.n_levels = d.n_levels;
    in.n_placements = (uint32_t)T.pl.size();
    in.n_states = (uint32_t)n_states;
    in.n_finals = (uint32_t)n_finals;
    in.fcr_s0 = d.fcr[0];
    in.full_mem_mib = d.full_mem;
    in.n_layout = d.n_layout;
    in.scheme_a = 1;
    for (uint32_t l = 0; l < d.n_levels; ++l)
        if (d.n_alay[l] == 0) in.scheme_a = 0;
    in.idle_w = idle_w;
    in.w_per_slice = wps;
    return MIG_OK;
}

}  // namespace

extern "C" {

mig_status mig_geometry_load(const char* path, mig_geometry** out) {
    if (!path || !out) return mig_set_error(MIG_E_INVALID_ARG, "mig_geometry_load: null argument");
    std::string p = path;
    if (p.rfind("builtin:", 0) == 0) {
        std::string name = p.substr(8);
        if (name.empty() || name.find('/') != std::string::npos)
            return mig_set_error(MIG_E_INVALID_ARG, "bad builtin geometry name");
        p = builtin_dir() + name + ".json";
    }
    std::string text;
    if (!read_file(p, &text)) return mig_set_error(MIG_E_IO, "cannot read geometry file " + p);
    mig_geometry* g = new mig_geometry();
    mig_status s = load_geometry(text, g);
    if (s != MIG_OK) {
        delete g;
        return s;
    }
    *out = g;
    return MIG_OK;
}

void mig_geometry_free(mig_geometry* g) { delete g; }

mig_status mig_geometry_query(const mig_geometry* g, mig_geometry_info* out) {
    if (!g || !out) return mig_set_error(MIG_E_INVALID_ARG, "mig_geometry_query: null argument");
    *out = g->info;
    return MIG_OK;
}

mig_status mig_geometry_profile(const mig_geometry* g, uint32_t p, uint32_t* mem_mib, uint32_t* compute,
                                uint32_t* slots, char name[32]) {
    if (!g) return mig_set_error(MIG_E_INVALID_ARG, "mig_geometry_profile: null geometry");
    if (p >= g->dg.n_prof) return mig_set_error(MIG_E_INVALID_ARG, "profile index out of range");
    if (mem_mib) *mem_mib = g->dg.mem[p];
    if (compute) *compute = g->dg.comp[p];
    if (slots) *slots = (uint32_t)__builtin_popcount(g->dg.lenmask[p]);
    if (name) snprintf(name, 32, "%s", g->prof_names[p].c_str());
    return MIG_OK;
}

mig_status mig_geometry_fcr(const mig_geometry* g, uint32_t occ, uint32_t* fcr) {
    if (!g || !fcr) return mig_set_error(MIG_E_INVALID_ARG, "mig_geometry_fcr: null argument");
    if (occ >= (1u << g->dg.n_slots)) return mig_set_error(MIG_E_INVALID_ARG, "occupancy mask out of range");
    *fcr = g->dg.fcr[occ];
    return MIG_OK;
}

mig_status mig_geometry_place(const mig_geometry* g, uint32_t occ, uint32_t profile, int32_t* start) {
    if (!g || !start) return mig_set_error(MIG_E_INVALID_ARG, "mig_geometry_place: null argument");
    if (profile >= g->dg.n_prof) return mig_set_error(MIG_E_INVALID_ARG, "profile index out of range");
    if (occ >= (1u << g->dg.n_slots) || g->dg.fcr[occ] == 0)
        return mig_set_error(MIG_E_INVALID_ARG, "occupancy mask is not a valid state");
    uint32_t best = 0;
    for (uint32_t k = 0; k < g->dg.n_place[profile]; ++k) {
        uint32_t pl = g->dg.place[profile][k], s = pl & 0xFF, mask = pl >> 8;
        if (occ & mask) continue;
        uint32_t score = ((uint32_t)g->dg.fcr[occ | mask] << 8) | s;
        if (score > best) best = score;
    }
    *start = best ? (int32_t)(best & 0xFF) : -1;
    return MIG_OK;
}

mig_status mig_geometry_fusion(const mig_geometry* g, uint32_t occ, uint32_t sm, uint32_t busy, uint32_t profile,
                               int32_t* start, uint32_t* destroyed) {
    if (!g || !start || !destroyed) return mig_set_error(MIG_E_INVALID_ARG, "mig_geometry_fusion: null argument");
    const DevGeom& d = g->dg;
    if (profile >= d.n_prof) return mig_set_error(MIG_E_INVALID_ARG, "profile index out of range");
    if (g->a7.empty()) return mig_set_error(MIG_E_UNSUPPORTED, "no slot-level tables for this geometry");
    const uint32_t key = (occ & 0xFFu) | ((sm & 0xFFu) << 8);
    if (occ > 0xFFu || sm > 0xFFu || g->trans_id[key] < 0)
        return mig_set_error(MIG_E_INVALID_ARG, "(occupancy, starts) is not a reachable partition state");
    uint32_t cm = 0, cbase = 0;
    for (uint32_t p = 0; p < profile; ++p) cbase += 1u << d.n_place[p];
    for (uint32_t k = 0; k < d.n_place[profile]; ++k)
        if (!((d.place[profile][k] >> 8) & busy)) cm |= 1u << k;
    const uint32_t* e = &g->a7[((size_t)g->trans_id[key] * g->n_a7 + cbase + cm) * 2];
    *start = e[0] ? (int32_t)(e[0] & 0xFFu) : -1;
    *destroyed = e[0] ? (e[1] & 0xFFu) : 0u;
    return MIG_OK;
}

}  // extern "C"
