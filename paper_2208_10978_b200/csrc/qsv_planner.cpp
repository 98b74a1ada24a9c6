// qsv_planner.cpp -- native fusion planner (see qsv_planner.h).
#include "qsv_planner.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <unordered_map>

namespace qsv {

namespace {

inline int popc64(uint64_t v) { return __builtin_popcountll(v); }

inline int highest_bit(uint64_t v) { return 63 - __builtin_clzll(v); }

// Local (tile) image of a physical mask: bit i of the result = bit pos[i] of mask.
inline uint32_t compress(uint64_t mask, const TileGeom &g)
{
    uint32_t out = 0;
    for (int i = 0; i < g.m; ++i)
        if ((mask >> g.pos[i]) & 1ull) out |= 1u << i;
    return out;
}

inline uint64_t tile_mask(const TileGeom &g)
{
    uint64_t t = 0;
    for (int i = 0; i < g.m; ++i) t |= 1ull << g.pos[i];
    return t;
}

inline int local_of(const TileGeom &g, int q)
{
    for (int i = 0; i < g.m; ++i)
        if (g.pos[i] == q) return i;
    return -1;
}

void choose_tile(int n, int &m, int &c)
{
    m = n < kMaxTileBits ? n : kMaxTileBits;
    if (const char *env_m = getenv("QSV_TILE_BITS"))  // experiment: smaller tiles (more CTAs)
        m = std::max(6, std::min(m, atoi(env_m)));
    if (m == n) {
        c = n;
    } else {
        const char *env_c = getenv("QSV_MIN_CONTIG");  // low contiguous tile bits (default 3: 128 B segments)
        c = env_c ? std::max(1, std::min(kMinContig, atoi(env_c))) : 3;
        if (c > m - 4) c = m - 4;
        if (c < 0) c = 0;
    }
}

// Tile = low c bits + hi bits, topped up with the lowest unused bits.
TileGeom make_geom(int n, int m, int c, uint64_t hi)
{
    TileGeom g;
    std::memset(&g, 0, sizeof(g));
    g.n = n;
    g.m = m;
    uint64_t t = (c >= 64 ? ~0ull : ((1ull << c) - 1ull)) | hi;
    for (int q = 0; popc64(t) < m && q < n; ++q) t |= 1ull << q;
    int k = 0;
    for (int q = 0; q < n; ++q)
        if ((t >> q) & 1ull) g.pos[k++] = q;
    int cc = 0;
    while (cc < m && g.pos[cc] == cc) ++cc;
    g.c = cc;
    g.ncomp = 0;
    for (int q = 0; q < n; ++q)
        if (!((t >> q) & 1ull)) g.comp[g.ncomp++] = q;
    return g;
}

// One Pauli rotation / string in symplectic form.
struct Sym {
    uint64_t a;  // flip bits x|y
    uint64_t b;  // sign bits y|z
};

inline bool anticommute(const Sym &p, const Sym &q)
{
    return ((popc64(p.a & q.b) + popc64(p.b & q.a)) & 1) != 0;
}

struct Item {
    bool rot = false;
    int gate = -1;            // gate index (gate items)
    std::vector<int> rots;    // indices into the rotation list (rot items)
    uint64_t supp = 0;        // all touched qubits
    uint64_t req = 0;         // qubits that must be tile-local
    uint64_t a_union = 0, b_union = 0;
    int cluster = -1;         // dense-fused gate cluster (index into ProgramTemplate::cfills)
    int cost = 2;             // FP64 work (complex FMAs per amplitude) -- bounds a pass
    int par = 8;              // parameter doubles (specialised passes hold them in 64 KiB __constant__)
    uint64_t last_z = 0;      // rot items: Z mask of the last rotation (a change starts another OP_GMAT)
};

// Parameter doubles of a gate (op_param_count of the op it becomes) and of a
// same-flip rotation group (one OP_GMAT table: 16 << (|f| - 1) doubles).
int gate_par(int kind);
int rot_par(uint64_t flip)
{
    const int w = popc64(flip);
    return (w >= 1 && w <= 4) ? (16 << (w - 1)) : 0;
}

// Parameter budget of one pass: a specialised pass keeps its matrices in
// 64 KiB of constant memory (jit_source rejects > 8192 doubles).
int pass_param_cap()
{
    const char *e = getenv("QSV_PASS_PARAM_CAP");
    return e ? std::max(1, atoi(e)) : 8192;
}

bool conflict(const Item &A, const Item &B, const std::vector<Rot> &R)
{
    if (!A.rot || !B.rot) return (A.supp & B.supp) != 0;
    if (((A.a_union & B.b_union) | (A.b_union & B.a_union)) == 0) return false;
    for (int i : A.rots) {
        const Sym p{R[i].x | R[i].y, R[i].y | R[i].z};
        for (int j : B.rots) {
            const Sym q{R[j].x | R[j].y, R[j].y | R[j].z};
            if (anticommute(p, q)) return true;
        }
    }
    return false;
}

struct Schedule {
    std::vector<std::vector<int>> pass_items;
    std::vector<uint64_t> pass_hi;
    std::vector<bool> pass_global;
    std::vector<int> pass_cost;
    std::vector<int> pass_par;
};

Schedule schedule(const std::vector<Item> &items, const std::vector<Rot> &R, int n, int m, int c)
{
    Schedule S;
    const uint64_t low = c >= 64 ? ~0ull : ((1ull << c) - 1ull);
    const int free_slots = m - c;
    std::vector<int> item_pass(items.size(), 0);
    // FP64 budget of one pass (complex FMAs per amplitude).  With the
    // lookahead scheduler fewer, heavier passes win (config 2: cap 48 -> 27
    // passes / 82 ms, 128 -> 16 passes / 75 ms, FP64-bound); the cap only
    // keeps specialised kernels from growing without bound.
    const char *env_cap = getenv("QSV_PASS_COST_CAP");
    const int cost_cap = env_cap ? std::max(1, atoi(env_cap)) : 128;
    const int par_cap = pass_param_cap();
    for (size_t i = 0; i < items.size(); ++i) {
        const Item &it = items[i];
        const uint64_t need = it.req & ~low;
        const bool fits = popc64(need) <= free_slots;
        int earliest = 0;
        const int last = (int)S.pass_items.size() - 1;
        for (size_t jj = i; jj-- > 0;) {
            if (item_pass[jj] <= earliest) continue;
            if (conflict(items[jj], it, R)) {
                earliest = std::max(earliest, item_pass[jj]);
                if (earliest == last) break;
            }
        }
        int placed = -1;
        if (fits) {
            for (int p = earliest; p <= last; ++p) {
                if (S.pass_global[p]) continue;
                if (popc64(S.pass_hi[p] | need) <= free_slots &&
                    (S.pass_cost[p] + it.cost <= cost_cap || it.cost == 0) &&
                    S.pass_par[p] + it.par <= par_cap) {
                    placed = p;
                    break;
                }
            }
        }
        if (placed < 0) {
            // a new pass at the end; a global pass must also come after every
            // conflicting item, which `earliest <= last` already guarantees.
            S.pass_items.emplace_back();
            S.pass_hi.push_back(0);
            S.pass_global.push_back(!fits);
            S.pass_cost.push_back(0);
            S.pass_par.push_back(0);
            placed = (int)S.pass_items.size() - 1;
        }
        S.pass_items[placed].push_back((int)i);
        S.pass_hi[placed] |= need;
        S.pass_cost[placed] += it.cost;
        S.pass_par[placed] += it.par;
        item_pass[i] = placed;
    }
    return S;
}

// Lookahead pass construction: passes are built one at a time; a pass opens
// with the earliest ready item (every conflicting earlier item scheduled) and
// then repeatedly takes, from a window of upcoming ready items, the one that
// grows the tile's high-bit set least -- commuting items (disjoint qubits /
// even symplectic product) are pulled forward past non-fitting ones, so
// passes fill with items that share tile bits instead of closing as soon as
// the next item in circuit order does not fit.
Schedule schedule_lookahead(const std::vector<Item> &items, const std::vector<Rot> &R, int m, int c,
                            int cost_cap, int window)
{
    Schedule S;
    const uint64_t low = c >= 64 ? ~0ull : ((1ull << c) - 1ull);
    const int free_slots = m - c;
    const int N = (int)items.size();
    std::vector<int> npend(N, 0);
    std::vector<std::vector<int>> succ(N);
    for (int i = 0; i < N; ++i)
        for (int j = 0; j < i; ++j)
            if (conflict(items[j], items[i], R)) {
                succ[j].push_back(i);
                ++npend[i];
            }
    std::vector<char> done(N, 0);
    int first = 0, left = N;
    // Fill one pass greedily from `seed`; with `undo` the changes are rolled
    // back and only the pass's (work, items) score is returned.
    std::vector<int> taken;
    const int par_cap = pass_param_cap();
    auto fill = [&](int seed, bool undo, uint64_t &hi, int &cost) {
        taken.clear();
        hi = 0;
        cost = 0;
        int par = 0;
        auto take = [&](int i) {
            done[i] = 1;
            taken.push_back(i);
            hi |= items[i].req & ~low;
            cost += items[i].cost;
            par += items[i].par;
            for (int k : succ[i]) --npend[k];
        };
        take(seed);
        if (popc64(items[seed].req & ~low) <= free_slots) {
            for (;;) {
                int best = -1, best_growth = 1 << 30;
                const int lim = std::min(N, first + window);
                for (int i = first; i < lim; ++i) {
                    if (done[i] || npend[i] != 0) continue;
                    const uint64_t need = items[i].req & ~low;
                    if (popc64(hi | need) > free_slots) continue;
                    if (items[i].cost != 0 && cost + items[i].cost > cost_cap) continue;
                    if (par + items[i].par > par_cap) continue;
                    const int growth = popc64(need & ~hi);
                    if (growth < best_growth) {
                        best_growth = growth;
                        best = i;
                        if (growth == 0) break;
                    }
                }
                if (best < 0) break;
                take(best);
            }
        }
        if (undo)
            for (int i : taken) {
                done[i] = 0;
                for (int k : succ[i]) ++npend[k];
            }
    };
    const char *env_seeds = getenv("QSV_SCHED_SEEDS");
    const int nseeds = env_seeds ? std::max(1, atoi(env_seeds)) : (N <= 4096 ? 8 : 1);
    while (left > 0) {
        while (first < N && done[first]) ++first;
        // candidate seeds: the first ready items; keep the one whose pass
        // carries the most work (then the most items)
        int cands[64], nc = 0;
        for (int i = first; i < N && nc < nseeds && nc < 64; ++i)
            if (!done[i] && npend[i] == 0) cands[nc++] = i;
        int start = nc ? cands[0] : first;  // a DAG always has a ready item
        if (nc > 1 && popc64(items[start].req & ~low) <= free_slots) {
            long best_score = -1;
            for (int k = 0; k < nc; ++k) {
                if (popc64(items[cands[k]].req & ~low) > free_slots) continue;
                uint64_t hi;
                int cost;
                fill(cands[k], true, hi, cost);
                const long score = (long)cost * 4096 + (long)taken.size();
                if (score > best_score) {
                    best_score = score;
                    start = cands[k];
                }
            }
        }
        const bool fits = popc64(items[start].req & ~low) <= free_slots;
        uint64_t hi;
        int cost;
        fill(start, false, hi, cost);
        S.pass_items.push_back(taken);
        S.pass_hi.push_back(hi);
        S.pass_global.push_back(!fits);
        S.pass_cost.push_back(cost);
        left -= (int)taken.size();
    }
    return S;
}

// Pattern match of circuit.py:271-281 `_evolution_gates` at position i.
bool match_block(const int32_t *kinds, const int32_t *qubits, int64_t N, int64_t i, Rot &out,
                 int64_t &len)
{
    // Qubit order is not required to be ascending (the reference emits
    // ascending order, circuit.py:271-281, but a relabelled circuit -- e.g. a
    // shard's local segment in distributed.py -- is not): the block is
    // exp(-i theta/2 P) whenever the basis qubits are distinct, the ladder is a
    // chain over distinct qubits and everything is mirrored exactly.
    int64_t j = i;
    int bq[64], bk[64], nb = 0;
    uint64_t bmask = 0;
    while (j < N && (kinds[j] == K_H || kinds[j] == K_HY)) {
        const int q = qubits[2 * j];
        if (((bmask >> q) & 1ull) || nb >= 64) break;
        bmask |= 1ull << q;
        bq[nb] = q;
        bk[nb] = kinds[j];
        ++nb;
        ++j;
    }
    int s[66], ns = 0;
    uint64_t smask = 0;
    while (j < N && kinds[j] == K_CNOT) {
        const int a = qubits[2 * j], b = qubits[2 * j + 1];
        if (ns == 0) {
            s[0] = a;
            s[1] = b;
            ns = 2;
            smask = (1ull << a) | (1ull << b);
        } else {
            if (a != s[ns - 1] || ((smask >> b) & 1ull) || ns >= 64) break;
            s[ns++] = b;
            smask |= 1ull << b;
        }
        ++j;
    }
    if (j >= N || kinds[j] != K_RZ) return false;
    const int rzq = qubits[2 * j];
    if (ns == 0) {
        s[0] = rzq;
        ns = 1;
    } else if (rzq != s[ns - 1]) {
        return false;
    }
    const int64_t rz_index = j;
    ++j;
    for (int k = ns - 2; k >= 0; --k) {
        if (j >= N || kinds[j] != K_CNOT || qubits[2 * j] != s[k] || qubits[2 * j + 1] != s[k + 1])
            return false;
        ++j;
    }
    for (int k = 0; k < nb; ++k) {
        if (j >= N || kinds[j] != bk[k] || qubits[2 * j] != bq[k]) return false;
        ++j;
    }
    uint64_t supp = 0;
    for (int k = 0; k < ns; ++k) supp |= 1ull << s[k];
    uint64_t x = 0, y = 0;
    for (int k = 0; k < nb; ++k) {
        const uint64_t bit = 1ull << bq[k];
        if (!(supp & bit)) return false;
        if (bk[k] == K_H) x |= bit;
        else y |= bit;
    }
    out.x = x;
    out.y = y;
    out.z = supp & ~x & ~y;
    out.src = (int)rz_index;
    len = j - i;
    return true;
}

void build_items_from_rots(const std::vector<Rot> &R, std::vector<Item> &items)
{
    for (size_t r = 0; r < R.size(); ++r) {
        const uint64_t a = R[r].x | R[r].y, b = R[r].y | R[r].z;
        if (!items.empty() && items.back().rot && items.back().a_union == a &&
            (items.back().req == a)) {
            Item &g = items.back();
            g.rots.push_back((int)r);
            g.b_union |= b;
            g.supp |= a | b;
            if (R[r].z != g.last_z) g.par += rot_par(a);  // a run of another sign mask: its own table
            g.last_z = R[r].z;
            continue;
        }
        Item it;
        it.rot = true;
        it.cost = 0;
        it.par = rot_par(a);
        it.last_z = R[r].z;
        it.rots.push_back((int)r);
        it.a_union = a;
        it.b_union = b;
        it.supp = a | b;
        it.req = a;
        items.push_back(std::move(it));
    }
}

int param_count(int kind)
{
    switch (kind) {
        case K_H: case K_HY: case K_RY: case K_U3: return 8;
        case K_RZ: return 4;
        case K_CU3: return 32;
        default: return 0;
    }
}

// FP64 work of a gate in complex multiply-adds per amplitude: dense 2x2 = 2,
// diagonal = 1, permutation = 0 (folded into the tile map), dense 4x4 = 4.
int gate_cost(int kind)
{
    switch (kind) {
        case K_X: case K_CNOT: case K_SWAP: return 0;
        case K_RZ: return 1;
        case K_CU3: return 4;
        default: return 2;
    }
}

int gate_par(int kind)
{
    switch (kind) {
        case K_X: case K_CNOT: case K_SWAP: return 0;
        case K_RZ: return 4;
        case K_CU3: return 32;
        default: return 8;
    }
}

// Dense gate fusion (north star (1), k <= 2): walk the items in order and
// grow clusters of consecutive gates confined to <= 2 qubits.  A gate joins
// the open clusters on its qubits when their union stays within 2 qubits;
// otherwise the clusters that would widen it are closed (emitted) first.
// A closed cluster becomes one dense 2x2 / 4x4 item when that is cheaper than
// its gates (e.g. U3 U3 CNOT U3 U3: 8 -> 4 complex FMAs per amplitude).
// Default width is 1 (runs of single-qubit gates): measured on B200, the
// 4x4 form is slower in the specialised passes than the m00-real U3 form it
// replaces (config-2: 103 vs 97 ms), so QSV_FUSE_QUBITS=2 is opt-in.
// Emitting at close time is order-safe: everything emitted while a cluster is
// open acts on disjoint qubits and commutes with it.
void fuse_clusters(std::vector<Item> &items, const int32_t *kinds, const int32_t *qubits,
                   ProgramTemplate &t)
{
    struct Open {
        std::vector<int> gates;
        uint64_t qs = 0;
        int cost = 0;
        bool live = false;
    };
    std::vector<Open> cl;
    const char *env_fuse = getenv("QSV_FUSE_QUBITS");  // 0 / 1 / 2 (default 1)
    const int max_q = env_fuse ? std::max(0, std::min(2, atoi(env_fuse))) : 1;
    int open_of[kMaxQubits];
    for (int q = 0; q < kMaxQubits; ++q) open_of[q] = -1;
    std::vector<Item> out;
    out.reserve(items.size());
    auto gate_item = [&](int gi) {
        Item it;
        it.gate = gi;
        uint64_t s = 1ull << qubits[2 * gi];
        if (qubits[2 * gi + 1] >= 0) s |= 1ull << qubits[2 * gi + 1];
        it.supp = s;
        it.req = s;
        it.cost = gate_cost(kinds[gi]);
        it.par = gate_par(kinds[gi]);
        return it;
    };
    auto close = [&](int ci) {
        Open &C = cl[ci];
        if (!C.live) return;
        C.live = false;
        for (int q = 0; q < kMaxQubits; ++q)
            if (((C.qs >> q) & 1ull) && open_of[q] == ci) open_of[q] = -1;
        const int nq = popc64(C.qs);
        const int fused_cost = nq == 2 ? 4 : 2;
        if (C.gates.size() >= 2 && C.cost > fused_cost) {
            ClusterFill cf;
            cf.offset = -1;
            cf.qa = 63 - __builtin_clzll(C.qs);
            cf.qb = nq == 2 ? __builtin_ctzll(C.qs) : -1;
            cf.gates = C.gates;
            t.n_fused_gates += (int64_t)C.gates.size();
            Item it;
            it.cluster = (int)t.cfills.size();
            it.supp = C.qs;
            it.req = C.qs;
            it.cost = fused_cost;
            it.par = nq == 2 ? 32 : 8;
            t.cfills.push_back(std::move(cf));
            out.push_back(std::move(it));
        } else {
            for (int gi : C.gates) out.push_back(gate_item(gi));
        }
    };
    auto close_touching = [&](uint64_t mask) {
        // close in creation order (deterministic)
        int ids[kMaxQubits], k = 0;
        for (int q = 0; q < kMaxQubits; ++q)
            if (((mask >> q) & 1ull) && open_of[q] >= 0) {
                bool dup = false;
                for (int j = 0; j < k; ++j) dup |= ids[j] == open_of[q];
                if (!dup) ids[k++] = open_of[q];
            }
        std::sort(ids, ids + k);
        for (int j = 0; j < k; ++j) close(ids[j]);
    };
    for (Item &it : items) {
        if (it.rot || it.gate < 0 || popc64(it.supp) > max_q) {
            close_touching(it.supp);
            out.push_back(std::move(it));
            continue;
        }
        const int gi = it.gate;
        const uint64_t Q = it.supp;
        // clusters on Q that carry a qubit outside Q cannot absorb a 2q gate
        int ids[2], k = 0;
        for (int q = 0; q < kMaxQubits; ++q)
            if (((Q >> q) & 1ull) && open_of[q] >= 0 && (k == 0 || ids[0] != open_of[q])) ids[k++] = open_of[q];
        uint64_t uni = Q;
        for (int j = 0; j < k; ++j) uni |= cl[ids[j]].qs;
        if (popc64(uni) > max_q) {
            for (int j = 0; j < k; ++j)
                if (cl[ids[j]].qs & ~Q) close(ids[j]);
            int kk = 0;
            for (int j = 0; j < k; ++j)
                if (cl[ids[j]].live) ids[kk++] = ids[j];
            k = kk;
        }
        int target;
        if (k == 0) {
            cl.emplace_back();
            target = (int)cl.size() - 1;
            cl[target].live = true;
        } else {
            target = std::min(ids[0], k > 1 ? ids[1] : ids[0]);
            if (k == 2) {  // merge the other (disjoint qubits: the two commute)
                const int other = ids[0] == target ? ids[1] : ids[0];
                Open &O = cl[other];
                cl[target].gates.insert(cl[target].gates.end(), O.gates.begin(), O.gates.end());
                cl[target].qs |= O.qs;
                cl[target].cost += O.cost;
                O.live = false;
                O.gates.clear();
            }
        }
        Open &T = cl[target];
        T.gates.push_back(gi);
        T.qs |= Q;
        T.cost += gate_cost(kinds[gi]);
        for (int q = 0; q < kMaxQubits; ++q)
            if ((T.qs >> q) & 1ull) open_of[q] = target;
    }
    for (size_t ci = 0; ci < cl.size(); ++ci) close((int)ci);
    items.swap(out);
}

// Structural phase deferral (see PhaseDefer): a U3 item whose next item on
// its qubit is a CNOT with that qubit as control, followed on that qubit by
// another U3 item.  Returns per-gate flags for emit_program.
void find_phase_defers(const std::vector<Item> &items, const int32_t *kinds, const int32_t *qubits,
                       int n, ProgramTemplate &t)
{
    const char *env = getenv("QSV_PHASE_DEFER");
    if (env && env[0] == '0') return;
    // per qubit: the item indices touching it, in order
    std::vector<std::vector<int>> on(n);
    for (int i = 0; i < (int)items.size(); ++i)
        for (int q = 0; q < n; ++q)
            if ((items[i].supp >> q) & 1ull) on[q].push_back(i);
    auto plain_u3 = [&](int it) {
        return items[it].gate >= 0 && items[it].cluster < 0 && !items[it].rot &&
               kinds[items[it].gate] == K_U3;
    };
    std::vector<char> is_src(items.size(), 0), is_dst(items.size(), 0);
    for (int q = 0; q < n; ++q) {
        const auto &v = on[q];
        for (size_t k = 0; k + 2 < v.size(); ++k) {
            const int a = v[k], x = v[k + 1], b = v[k + 2];
            if (!plain_u3(a) || !plain_u3(b)) continue;
            const Item &cx = items[x];
            if (cx.gate < 0 || cx.cluster >= 0 || kinds[cx.gate] != K_CNOT || qubits[2 * cx.gate] != q)
                continue;
            if (is_src[a]) continue;
            is_src[a] = 1;
            is_dst[b] = 1;
            t.defers.push_back(PhaseDefer{items[a].gate, items[b].gate});
        }
    }
}

// The control qubit of a CzDefer's OP_U1C: the qubit of its source U3.
inline int czdefer_target_qubit(const CzDefer &d, const int32_t *qubits) { return qubits[2 * d.src]; }

// Controlled-phase deferrals (see CzDefer): for a CNOT(c, t) item between a
// plain U3 G on t (not a PhaseDefer source) and plain U3s T (next on t) and K
// (next on c, not a deferral source, K before T in item order), G's phase
// goes to T, to K, and to K's control-selected copy; K then also requires t
// (its control) in registers and must run before T, which the added support
// bit enforces in every scheduler (items sharing a qubit are ordered).
void find_cz_defers(std::vector<Item> &items, const int32_t *kinds, const int32_t *qubits, int n,
                    int m, ProgramTemplate &t)
{
    const char *env = getenv("QSV_CZ_DEFER");
    if ((env && env[0] == '0') || m < kBlockBits + 1) return;
    std::vector<std::vector<int>> on(n);
    for (int i = 0; i < (int)items.size(); ++i)
        for (int q = 0; q < n; ++q)
            if ((items[i].supp >> q) & 1ull) on[q].push_back(i);
    auto plain_u3 = [&](int it) {
        return it >= 0 && items[it].gate >= 0 && items[it].cluster < 0 && !items[it].rot &&
               kinds[items[it].gate] == K_U3;
    };
    std::unordered_map<int, char> pd_src;  // gate -> PhaseDefer source
    for (const PhaseDefer &d : t.defers) pd_src[d.src] = 1;
    std::vector<char> cz_src(items.size(), 0), cz_ctl(items.size(), 0);
    auto pos_in = [](const std::vector<int> &v, int x) {
        for (size_t k = 0; k < v.size(); ++k)
            if (v[k] == x) return (int)k;
        return -1;
    };
    for (int x = 0; x < (int)items.size(); ++x) {
        const Item &cx = items[x];
        if (cx.gate < 0 || cx.cluster >= 0 || cx.rot || kinds[cx.gate] != K_CNOT) continue;
        const int c = qubits[2 * cx.gate], tq = qubits[2 * cx.gate + 1];
        const int pt = pos_in(on[tq], x), pc = pos_in(on[c], x);
        if (pt < 1 || pt + 1 >= (int)on[tq].size() || pc < 0 || pc + 1 >= (int)on[c].size()) continue;
        const int G = on[tq][pt - 1], T = on[tq][pt + 1], K = on[c][pc + 1];
        if (!plain_u3(G) || !plain_u3(T) || !plain_u3(K) || K >= T) continue;
        if (pd_src.count(items[G].gate) || pd_src.count(items[K].gate)) continue;
        if (cz_src[G] || cz_ctl[G] || cz_src[K] || cz_ctl[K]) continue;
        cz_src[G] = 1;
        cz_ctl[K] = 1;
        items[K].supp |= 1ull << tq;
        items[K].req |= 1ull << tq;
        items[K].par = 16;
        t.czdefers.push_back(CzDefer{items[G].gate, items[T].gate, items[K].gate});
    }
}

// Fixed 2x2 / 4x4 matrices of the permutation gates (circuit.py:36-45).
void perm_matrix(int kind, double *o)
{
    const int n = kind == K_X ? 2 : 4;
    for (int i = 0; i < 2 * n * n; ++i) o[i] = 0.0;
    auto one = [&](int r, int c) { o[2 * (r * n + c)] = 1.0; };
    if (kind == K_X) { one(0, 1); one(1, 0); }
    else if (kind == K_CNOT) { one(0, 0); one(1, 1); one(2, 3); one(3, 2); }
    else { one(0, 0); one(1, 2); one(2, 1); one(3, 3); }
}

void cluster_matrix(const ClusterFill &cf, const int32_t *kinds, const int32_t *qubits,
                    const double *values, double *out)
{
    const int n = cf.qb >= 0 ? 4 : 2;
    double M[32], G[32], N[32], g[32];
    for (int i = 0; i < 2 * n * n; ++i) M[i] = 0.0;
    for (int i = 0; i < n; ++i) M[2 * (i * n + i)] = 1.0;
    for (int gi : cf.gates) {
        const int kind = kinds[gi];
        const int q0 = qubits[2 * gi], q1 = qubits[2 * gi + 1];
        if (kind == K_X || kind == K_CNOT || kind == K_SWAP) perm_matrix(kind, g);
        else gate_matrix(kind, values + 3 * (size_t)gi, g);
        if (kind == K_RZ) {  // diag(d0, d1) -> dense 2x2
            const double d0r = g[0], d0i = g[1], d1r = g[2], d1i = g[3];
            for (int i = 0; i < 8; ++i) g[i] = 0.0;
            g[0] = d0r; g[1] = d0i; g[6] = d1r; g[7] = d1i;
        }
        for (int i = 0; i < 2 * n * n; ++i) G[i] = 0.0;
        const bool two = q1 >= 0;
        if (n == 2) {
            for (int i = 0; i < 8; ++i) G[i] = g[i];
        } else if (!two) {
            // 1q gate on qa (MSB, bit 1 of the 4x4 index) or qb (bit 0)
            const int sh = q0 == cf.qa ? 1 : 0;
            for (int r = 0; r < 4; ++r)
                for (int c = 0; c < 4; ++c) {
                    const int other = 1 - sh;
                    if (((r >> other) & 1) != ((c >> other) & 1)) continue;
                    const int rr = (r >> sh) & 1, cc = (c >> sh) & 1;
                    G[2 * (r * 4 + c)] = g[2 * (rr * 2 + cc)];
                    G[2 * (r * 4 + c) + 1] = g[2 * (rr * 2 + cc) + 1];
                }
        } else {
            // 4x4 in (bit q0, bit q1) order; re-index to (bit qa, bit qb)
            const bool same = q0 == cf.qa;
            auto idx = [&](int r) { return same ? r : ((r & 1) << 1) | (r >> 1); };
            for (int r = 0; r < 4; ++r)
                for (int c = 0; c < 4; ++c) {
                    G[2 * (r * 4 + c)] = g[2 * (idx(r) * 4 + idx(c))];
                    G[2 * (r * 4 + c) + 1] = g[2 * (idx(r) * 4 + idx(c)) + 1];
                }
        }
        for (int r = 0; r < n; ++r)
            for (int c = 0; c < n; ++c) {
                double re = 0, im = 0;
                for (int l = 0; l < n; ++l) {
                    const double ar = G[2 * (r * n + l)], ai = G[2 * (r * n + l) + 1];
                    const double br = M[2 * (l * n + c)], bi = M[2 * (l * n + c) + 1];
                    re += ar * br - ai * bi;
                    im += ar * bi + ai * br;
                }
                N[2 * (r * n + c)] = re;
                N[2 * (r * n + c) + 1] = im;
            }
        for (int i = 0; i < 2 * n * n; ++i) M[i] = N[i];
    }
    for (int i = 0; i < 2 * n * n; ++i) out[i] = M[i];
}

void block_pass(ProgramTemplate &t, PassPlan &pp);

// U3Norm.  A U3 (FP64-bound brickwork) costs 14 FP64 instructions per pair
// (12 phase-deferred).  Dividing the gate by a real scalar changes only a
// global factor, and the factors of one pass are multiplied back into ONE of
// its gates (the sink), so the pass's output is exact:
//   mode 4: U3 / c, c = cos(theta/2): m00 = 1 -> row 0 is 2 DFMA per
//           component: 12 per pair;
//   mode 6 (phase-deferring U3, see PhaseDefer):
//           U3(t, 0, l) = c diag(1, e^{il}) [[1, -e^{il} tan], [e^{-il} tan, 1]]
//           -- the diag(1, e^{il}) is deferred with the phi phase (it commutes
//           with the CNOT control and lands in the next U3's lambda), the
//           shear costs 8 per pair.
// Brickwork (config 2): 12.7 -> ~10 FP64 instructions per pair per U3.  An
// angle with |cos(theta/2)| < 1e-3 sends the call to a plan without the
// normalised forms (set_plain_u3), so tan never blows up.
void assign_u3_norm(ProgramTemplate &t, const PassPlan &pp, int pass, const int32_t *kinds)
{
    if ((int)t.pass_sink.size() <= pass) t.pass_sink.resize(pass + 1, -1);
    if (t.fill_mode.size() < t.fills.size()) {
        t.fill_mode.resize(t.fills.size(), 0);
        t.fill_pass.resize(t.fills.size(), -1);
    }
    const char *env = getenv("QSV_U3_NORM");
    if (plain_u3() || (env && env[0] == '0')) return;
    // the pass's plain U3 ops and their fills
    std::vector<std::pair<int, int>> u3;  // (op index, fill index)
    for (int k = pp.op_begin; k < pp.op_end; ++k) {
        const OpRec &op = t.ops[k];
        if ((op.type != OP_U1 && op.type != OP_U1C) || op.p < 0) continue;
        for (size_t f = 0; f < t.fills.size(); ++f)
            if (t.fills[f].offset == op.p && t.fills[f].kind == K_U3) {
                u3.push_back({k, (int)f});
                break;
            }
    }
    if (u3.size() < 2) return;
    // sink: a plain non-deferring U3 if there is one (it loses 2 of 14, a
    // deferring one 4 of 12); a controlled one only as the last resort
    size_t sink = u3.size();
    for (size_t i = 0; i < u3.size() && sink == u3.size(); ++i)
        if (t.ops[u3[i].first].h != 3 && t.ops[u3[i].first].type == OP_U1) sink = i;
    for (size_t i = 0; i < u3.size() && sink == u3.size(); ++i)
        if (t.ops[u3[i].first].type == OP_U1) sink = i;
    if (sink == u3.size()) sink = 0;
    t.pass_sink[pass] = u3[sink].second;
    for (size_t i = 0; i < u3.size(); ++i) {
        t.fill_pass[u3[i].second] = pass;
        if (i == sink) continue;
        OpRec &op = t.ops[u3[i].first];
        const int mode = op.h == 3 ? 6 : 4;
        op.h = mode;
        t.fill_mode[u3[i].second] = (int8_t)mode;
    }
    (void)kinds;
}

void emit_program(int n, int m, int c, const std::vector<Item> &items, const std::vector<Rot> &R,
                  const int32_t *kinds, const int32_t *qubits, const Schedule &S,
                  ProgramTemplate &t)
{
    t.n = n;
    t.m = m;
    t.c = c;
    for (size_t p = 0; p < S.pass_items.size(); ++p) {
        PassPlan pp;
        if (S.pass_global[p]) {
            // single rotation group, applied over the whole state
            std::memset(&pp.geom, 0, sizeof(pp.geom));
            pp.geom.n = n;
            pp.global = true;
            pp.op_begin = (int)t.ops.size();
            for (int ii : S.pass_items[p]) {
                const Item &it = items[ii];
                OpRec op{};
                op.type = OP_ROTG;
                op.r0 = (int)t.rots.size();
                for (int r : it.rots) {
                    RotRec rr{};
                    rr.s_hi = R[r].y | R[r].z;
                    rr.s_loc = 0;
                    const int ny = popc64(R[r].y);
                    rr.q = ((ny + 3) & 3) | ((ny & 1) << 2);
                    t.rots.push_back(rr);
                    t.rot_src.push_back(R[r].src);
                }
                op.r1 = (int)t.rots.size();
                pp.flip = it.a_union;
                t.ops.push_back(op);
            }
            pp.op_end = (int)t.ops.size();
            t.passes.push_back(pp);
            ++t.n_fallback;
            continue;
        }
        pp.geom = make_geom(n, m, c, S.pass_hi[p]);
        const TileGeom &g = pp.geom;
        const uint64_t tm = tile_mask(g);
        pp.op_begin = (int)t.ops.size();
        for (int ii : S.pass_items[p]) {
            const Item &it = items[ii];
            OpRec op{};
            if (it.rot) {
                const uint64_t a = it.a_union;
                op.r0 = (int)t.rots.size();
                for (int r : it.rots) {
                    RotRec rr{};
                    const uint64_t b = R[r].y | R[r].z;
                    rr.s_hi = b & ~tm;
                    rr.s_loc = compress(b, g);
                    const int ny = popc64(R[r].y);
                    rr.q = ((ny + 3) & 3) | ((ny & 1) << 2);
                    t.rots.push_back(rr);
                    t.rot_src.push_back(R[r].src);
                }
                op.r1 = (int)t.rots.size();
                if (a == 0) {
                    op.type = OP_ROTD;
                } else {
                    op.type = OP_ROTG;
                    op.f = compress(a, g);
                    op.h = highest_bit(op.f);
                }
            } else if (it.cluster >= 0) {
                ClusterFill &cf = t.cfills[it.cluster];
                op.a = local_of(g, cf.qa);
                op.b = cf.qb >= 0 ? local_of(g, cf.qb) : -1;
                op.type = cf.qb >= 0 ? OP_U2 : OP_U1;
                op.p = (int)t.n_params;
                cf.offset = (int)t.n_params;
                t.n_params += cf.qb >= 0 ? 32 : 8;
            } else {
                const int gi = it.gate, kind = kinds[gi];
                const int a = local_of(g, qubits[2 * gi]);
                const int b = (kind == K_CNOT || kind == K_SWAP || kind == K_CU3)
                                  ? local_of(g, qubits[2 * gi + 1])
                                  : -1;
                op.a = a;
                op.b = b;
                switch (kind) {
                    case K_X: op.type = OP_X; break;
                    case K_CNOT: op.type = OP_CX; break;
                    case K_SWAP: op.type = OP_SWAP; break;
                    case K_RZ: op.type = OP_DIAG1; break;
                    case K_CU3: op.type = OP_U2; break;
                    default: op.type = OP_U1; break;
                }
                int ctrl = 0;
                if (kind == K_U3)
                    for (const CzDefer &d : t.czdefers)
                        if (d.ctl == gi) {
                            // controlled by the CNOT target of the deferral
                            int tq = -1;
                            for (const CzDefer &e : t.czdefers)
                                if (e.ctl == gi) tq = czdefer_target_qubit(e, qubits);
                            op.type = OP_U1C;
                            op.b = local_of(g, tq);
                            ctrl = 1;
                            break;
                        }
                // matrix class of a U1 (lets specialised passes drop zero
                // imaginary parts): 2 = all entries real (H, RY),
                // 1 = m00 real (U3: m00 = cos(theta/2); HY)
                if (op.type == OP_U1 || op.type == OP_U1C)
                    op.h = (kind == K_H || kind == K_RY) ? 2 : (kind == K_U3 || kind == K_HY) ? 1 : 0;
                if (op.type == OP_U1 && kind == K_U3) {
                    for (const PhaseDefer &d : t.defers)
                        if (d.src == gi) op.h = 3;  // V: m00 and m10 real
                    for (const CzDefer &d : t.czdefers)
                        if (d.src == gi) op.h = 3;  // V too: its phase is deferred
                }
                const int np = ctrl ? 16 : param_count(kind);
                if (np) {
                    op.p = (int)t.n_params;
                    t.fills.push_back(ParamFill{(int)t.n_params, gi, kind, ctrl});
                    t.n_params += np;
                }
            }
            t.ops.push_back(op);
        }
        pp.op_end = (int)t.ops.size();
        assign_u3_norm(t, pp, (int)t.passes.size(), kinds);
        if (g.m >= kBlockBits + 1) block_pass(t, pp);
        t.passes.push_back(pp);
    }
    t.n_items = (int64_t)items.size();
}

inline uint16_t swz16(uint32_t l) { return (uint16_t)tile_swz(l); }

// Group a pass's tile-local ops into register blocks of <= 4 logical tile
// bits, fold the permutation gates (CNOT / SWAP / X) into the pass's
// GF(2)-affine SMEM map, and rewrite ops to the block encoding (see BlockRec).
void block_pass(ProgramTemplate &t, PassPlan &pp)
{
    const int m = pp.geom.m;
    std::vector<OpRec> src(t.ops.begin() + pp.op_begin, t.ops.begin() + pp.op_end);
    std::vector<OpRec> out;
    pp.block_begin = (int)t.blocks.size();
    uint32_t A[12];   // map columns (unswizzled slot vectors) of the logical tile bits
    uint32_t tr = 0;  // map translation
    for (int b = 0; b < 12; ++b) A[b] = 1u << b;
    auto is_perm = [](int type) { return type == OP_CX || type == OP_SWAP || type == OP_X; };
    auto rot_signs = [&](const OpRec &op) {
        uint32_t u = 0;
        for (int r = op.r0; r < op.r1; ++r) u |= t.rots[r].s_loc;
        return u;
    };
    auto supp = [&](const OpRec &op) -> uint32_t {
        switch (op.type) {
            case OP_U1: case OP_X: case OP_DIAG1: return 1u << op.a;
            case OP_U2: case OP_U1C: case OP_CX: case OP_SWAP: return (1u << op.a) | (1u << op.b);
            case OP_ROTG: return op.f | rot_signs(op);
            case OP_ROTD: return rot_signs(op);
            default: return 0u;
        }
    };
    auto req = [](const OpRec &op) -> uint32_t {
        switch (op.type) {
            case OP_U1: return 1u << op.a;
            case OP_U2: case OP_U1C: return (1u << op.a) | (1u << op.b);
            case OP_ROTG: return op.f;
            default: return 0u;  // diagonal ops fit any block
        }
    };
    // Warp-local block transitions: three tile bits W are kept as the warp
    // index bits (thread bits 5-7) of every block whose register bits avoid
    // them.  Consecutive such blocks then read and write the same W-coset of
    // slots per warp (a permutation between them must not move W bits), so
    // the transition needs only __syncwarp instead of a group barrier --
    // warps run ahead of each other through chains of blocks.  W = the three
    // tile bits fewest ops need in registers.
    uint32_t Wmask = 0;
    bool has_rot = false;
    for (const OpRec &op : src) has_rot |= op.type == OP_ROTG || op.type == OP_ROTD;
    // (measured: a gain on gate passes, a loss on rotation-group passes,
    // where the fixed warp bits cost bank-conflict-free coset orders)
    if (m == kMaxTileBits && kBlockBits == 4 && !has_rot) {
        int cnt[12] = {0};
        for (const OpRec &op : src)
            if (op.type == OP_U1 || op.type == OP_U2 || op.type == OP_U1C || op.type == OP_ROTG)
                for (int b = 0; b < m; ++b) cnt[b] += (req(op) >> b) & 1u;
        for (int k = 0; k < 3; ++k) {
            int best = -1;
            for (int b = m - 1; b >= 0; --b)
                if (!((Wmask >> b) & 1u) && (best < 0 || cnt[b] < cnt[best])) best = b;
            Wmask |= 1u << best;
        }
        const char *env_wl = getenv("QSV_WARP_LOCAL");
        if (env_wl && env_wl[0] == '0') Wmask = 0;
    }
    bool prev_conform = false, perm_breaks = false;
    auto apply_perm = [&](const OpRec &op) {
        // psi'(L) = psi(P L) with P an involution, data unmoved: map' = map o P
        if (op.type == OP_CX) A[op.a] ^= A[op.b];
        else if (op.type == OP_SWAP) std::swap(A[op.a], A[op.b]);
        else tr ^= A[op.a];
        // does P move W bits (map a warp's W-coset onto another)?
        const uint32_t moved = op.type == OP_CX ? (1u << op.b)
                               : op.type == OP_SWAP ? ((1u << op.a) | (1u << op.b))
                                                    : (1u << op.a);
        if (moved & Wmask) perm_breaks = true;
    };
    std::vector<OpRec> pending, perms;
    uint32_t cur = 0, D = 0;
    uint32_t Ab[12], tb = 0;  // map at block start
    auto start_block = [&]() {
        std::copy(A, A + 12, Ab);
        tb = tr;
    };
    auto flush = [&]() {
        if (!pending.empty()) {
            constexpr int RB = kBlockBits, TB = kMaxTileBits - kBlockBits;
            bool conform = Wmask != 0 && (cur & Wmask) == 0;
            // The filler register bits (beyond the ones the ops need) are free:
            // if the default ones leave the lane-eligible thread columns (not
            // in registers, not W bits of a conforming block) without three
            // independent granule vectors, every LDS/STS of the block is a
            // 2-way bank conflict -- pick fillers that keep the rank at 3, or
            // else give up the warp-local W placement for this block (a group
            // barrier instead of __syncwarp around it).
            auto lane_rank = [&](uint32_t regs, bool conf) {
                uint32_t basis[3] = {0, 0, 0};
                int np = 0;
                for (int b = 0; b < m && np < 3; ++b) {
                    if (((regs >> b) & 1u) || (conf && ((Wmask >> b) & 1u))) continue;
                    uint32_t v = swz16(Ab[b]) & 7u;
                    for (int j = 0; j < np; ++j)
                        if ((v ^ basis[j]) < v) v ^= basis[j];
                    if (v == 0) continue;
                    basis[np] = v;
                    for (int a = np; a > 0 && basis[a] > basis[a - 1]; --a) std::swap(basis[a], basis[a - 1]);
                    ++np;
                }
                return np;
            };
            auto fill = [&](bool conf) {
                uint32_t regs = cur;
                for (int b = m - 1; b >= 0 && __builtin_popcount(regs) < RB; --b)
                    if (!conf || !((Wmask >> b) & 1u)) regs |= 1u << b;
                if (lane_rank(regs, conf) == 3) return regs;
                int cand[12], nc = 0;  // filler candidates, preferred (high) bits first
                for (int b = m - 1; b >= 0; --b)
                    if (!((cur >> b) & 1u) && (!conf || !((Wmask >> b) & 1u))) cand[nc++] = b;
                const int need = RB - __builtin_popcount(cur);
                for (uint32_t sel = 0; sel < (1u << nc); ++sel) {
                    if (__builtin_popcount(sel) != need) continue;
                    uint32_t alt = cur;
                    for (int i = 0; i < nc; ++i)
                        if ((sel >> i) & 1u) alt |= 1u << cand[i];
                    if (lane_rank(alt, conf) == 3) return alt;
                }
                return regs;
            };
            uint32_t bits = fill(conform);
            if (conform && lane_rank(bits, true) < 3) {
                const uint32_t alt = fill(false);
                if (lane_rank(alt, false) == 3) {
                    bits = alt;
                    conform = false;
                }
            }
            int pos[RB], nb[12], k = 0, kn = 0;
            for (int b = 0; b < m; ++b) {
                if ((bits >> b) & 1u) pos[k++] = b;
                else nb[kn++] = b;
            }
            // Thread bits 0-2 index the 8 lanes of a quarter warp, whose 16 B
            // LDS/STS must land in 8 distinct granules of a 128 B bank row:
            // put first three non-block bits whose swizzled slot columns are
            // independent in their granule bits (low 3 bits).  Any order of
            // the thread bits is valid -- gather, scatter and the per-block
            // sign / thread-bit tables all use this same nb[] order.
            // conforming blocks: the W bits go last (thread bits 5-7)
            int kl = kn;  // leading (lane + low thread) bits eligible for reordering
            if (conform) {
                int lead[12], tail[12], nl = 0, nt = 0;
                for (int i = 0; i < kn; ++i) {
                    if ((Wmask >> nb[i]) & 1u) tail[nt++] = nb[i];
                    else lead[nl++] = nb[i];
                }
                for (int i = 0; i < nl; ++i) nb[i] = lead[i];
                for (int i = 0; i < nt; ++i) nb[nl + i] = tail[i];
                kl = nl;
            }
            if (kl >= 3) {
                int pick[3], np = 0;
                uint32_t basis[3] = {0, 0, 0};  // reduced granule vectors
                for (int i = 0; i < kl && np < 3; ++i) {
                    uint32_t v = swz16(Ab[nb[i]]) & 7u;
                    for (int j = 0; j < np; ++j)
                        if ((v ^ basis[j]) < v) v ^= basis[j];
                    if (v == 0) continue;
                    // keep the basis in echelon form (distinct leading bits)
                    basis[np] = v;
                    for (int a = np; a > 0 && basis[a] > basis[a - 1]; --a) std::swap(basis[a], basis[a - 1]);
                    pick[np++] = i;
                }
                if (np == 3) {
                    int reordered[12], r = 0;
                    for (int j = 0; j < 3; ++j) reordered[r++] = nb[pick[j]];
                    for (int i = 0; i < kl; ++i)
                        if (i != pick[0] && i != pick[1] && i != pick[2]) reordered[r++] = nb[i];
                    for (int i = 0; i < kl; ++i) nb[i] = reordered[i];
                }
            }
            auto local = [&](int b) {
                for (int j = 0; j < RB; ++j)
                    if (pos[j] == b) return j;
                return -1;
            };
            auto thread_index = [&](int b) {
                for (int i = 0; i < kn; ++i)
                    if (nb[i] == b) return i;
                return -1;
            };
            auto comp_b = [&](uint32_t mask) {
                uint32_t o = 0;
                for (int j = 0; j < RB; ++j)
                    if ((mask >> pos[j]) & 1u) o |= 1u << j;
                return o;
            };
            auto expand_b = [&](uint32_t loc) {
                uint32_t o = 0;
                for (int j = 0; j < RB; ++j)
                    if ((loc >> j) & 1u) o |= 1u << pos[j];
                return o;
            };
            auto comp_t = [&](uint32_t mask) {
                uint32_t o = 0;
                for (int i = 0; i < kn; ++i)
                    if ((mask >> nb[i]) & 1u) o |= 1u << i;
                return o;
            };
            BlockRec br{};
            br.kind = 0;
            // entry flag: the transition into this block may be __syncwarp
            br.pad0 = (prev_conform && conform && !perm_breaks) ? 1 : 0;
            prev_conform = conform;
            perm_breaks = false;
            for (int i = 0; i < kn && i < TB; ++i) br.cols[i] = swz16(Ab[nb[i]]);
            for (int j = 0; j < RB; ++j) br.cols[TB + j] = swz16(Ab[pos[j]]);
            br.tswz = swz16(tb);
            br.op0 = (int)out.size();
            for (OpRec op : pending) {
                switch (op.type) {
                    case OP_U1: op.a = local(op.a); break;
                    case OP_U2: case OP_U1C: op.a = local(op.a); op.b = local(op.b); break;
                    case OP_DIAG1: {
                        const int j = local(op.a);
                        op.b = j >= 0 ? 0 : thread_index(op.a);
                        op.a = j;
                        break;
                    }
                    case OP_ROTG: op.f = comp_b(op.f); break;
                    case OP_CX: case OP_SWAP: op.a = local(op.a); op.b = local(op.b); break;
                    case OP_X: op.a = local(op.a); break;
                    default: break;
                }
                if (op.type == OP_ROTG || op.type == OP_ROTD)
                    for (int r = op.r0; r < op.r1; ++r)
                        t.rots[r].q = (t.rots[r].q & 0xff) | (int32_t)(comp_b(t.rots[r].s_loc) << 8) |
                                      (int32_t)(comp_t(t.rots[r].s_loc) << 12);
                if (op.type == OP_ROTG) {
                    // fuse each run of strings that share the sign bits off the
                    // flip (the JW Z-chain of one excitation): one 2x2 per pair
                    // per run instead of one per rotation -- and a form the
                    // specialised passes have (a lone rotation is a run of one)
                    const uint32_t fl = expand_b(op.f);
                    int r = op.r0;
                    while (r < op.r1) {
                        const uint32_t zc = t.rots[r].s_loc & ~fl;
                        const uint64_t zh = t.rots[r].s_hi;
                        int e = r + 1;
                        while (e < op.r1 && (t.rots[e].s_loc & ~fl) == zc && t.rots[e].s_hi == zh) ++e;
                        GmatFill gf;
                        gf.r0 = r;
                        gf.r1 = e;
                        gf.F = (int)op.f;
                        gf.H = 31 - __builtin_clz(op.f);
                        gf.w = __builtin_popcount(op.f);
                        for (int k = r; k < e; ++k) gf.yF.push_back((uint8_t)comp_b(t.rots[k].s_loc & fl));
                        gf.offset = (int)t.n_params;
                        t.n_params += (size_t)8 * (2u << (gf.w - 1));
                        t.gfills.push_back(gf);
                        // common masks live in a dedicated record
                        RotRec cr = t.rots[r];
                        cr.q = (int32_t)(comp_b(zc) << 8) | (int32_t)(comp_t(zc) << 12);
                        cr.s_loc = zc;
                        t.rots.push_back(cr);
                        t.rot_src.push_back(t.rot_src[r]);
                        OpRec g = op;
                        g.type = OP_GMAT;
                        g.p = gf.offset;
                        g.r0 = (int)t.rots.size() - 1;
                        g.r1 = g.r0 + 1;
                        out.push_back(g);
                        r = e;
                    }
                    continue;
                }
                out.push_back(op);
            }
            br.op1 = (int)out.size();
            t.blocks.push_back(br);
        }
        for (const OpRec &op : perms) apply_perm(op);
        pending.clear();
        perms.clear();
        cur = 0;
        D = 0;
    };
    // Partitioned block order: cut the tile's bits into fixed groups of 4
    // adjacent bits and emit, group after group, every op that is ready (its
    // predecessors on shared bits emitted) and confined to the group; ops
    // spanning groups (brickwork CNOTs across a cut) are emitted between
    // clusters, where a permutation only changes the SMEM map.  A brickwork
    // pass then needs ~one register block per group per two layers instead
    // of one per layer.  Order-safe: ops sharing a bit keep their order.
    std::vector<char> cluster_start;
    const char *env_part = getenv("QSV_BLOCK_PARTITION");
    if (!(env_part && env_part[0] == '0') && src.size() > 2 && m >= 8) {
        const int N = (int)src.size();
        std::vector<uint32_t> sp(N), rq(N);
        for (int i = 0; i < N; ++i) {
            sp[i] = supp(src[i]);
            rq[i] = is_perm(src[i].type) ? sp[i] : req(src[i]);
        }
        std::vector<int> npred(N, 0);
        std::vector<std::vector<int>> succ(N);
        for (int i = 0; i < N; ++i)
            for (int j = 0; j < i; ++j)
                if ((sp[i] & sp[j]) || (sp[i] == 0 && sp[j] == 0)) {
                    succ[j].push_back(i);
                    ++npred[i];
                }
        // candidate partitions: groups of 4 consecutive bits starting at
        // offset 0..3 (the first group takes the bits below the offset)
        auto build_order = [&](int shift, std::vector<OpRec> &order, std::vector<char> &starts) {
            std::vector<int> np = npred;
            std::vector<char> done(N, 0);
            order.clear();
            order.reserve(N);
            starts.assign(N, 0);
            int left = N;
            auto emit = [&](int i, bool start) {
                starts[order.size()] = start ? 1 : 0;
                done[i] = 1;
                --left;
                order.push_back(src[i]);
                for (int k : succ[i]) --np[k];
            };
            std::vector<uint32_t> groups;
            uint32_t g0 = (1u << shift) - 1u;
            for (int b = shift; b < m; b += kBlockBits) {
                uint32_t G = (((1u << kBlockBits) - 1u) << b) & ((1u << m) - 1u);
                if (g0) {
                    G |= g0;  // may exceed 4 bits: split below
                    g0 = 0;
                }
                if (__builtin_popcount(G) > kBlockBits) {
                    groups.push_back(G & ((1u << shift) - 1u));
                    G &= ~((1u << shift) - 1u);
                }
                if (G) groups.push_back(G);
            }
            while (left > 0) {
                bool progress = false;
                for (uint32_t G : groups) {
                    bool first = true;
                    for (bool more = true; more;) {
                        more = false;
                        for (int i = 0; i < N; ++i)
                            if (!done[i] && np[i] == 0 && rq[i] != 0 && (rq[i] & ~G) == 0) {
                                emit(i, first);
                                first = false;
                                more = progress = true;
                            }
                    }
                }
                for (int i = 0; i < N; ++i)
                    if (!done[i] && np[i] == 0) {
                        bool inside = false;
                        for (uint32_t G : groups)
                            if (rq[i] != 0 && (rq[i] & ~G) == 0) inside = true;
                        if (inside) continue;
                        emit(i, true);
                        progress = true;
                    }
                if (!progress)
                    for (int i = 0; i < N; ++i)
                        if (!done[i] && np[i] == 0) {
                            emit(i, true);
                            break;
                        }
            }
        };
        std::vector<OpRec> order, cand;
        std::vector<char> cand_starts;
        // keep the partitioned order only if it yields fewer register blocks
        // (dry run of the block former below: same flush rules, no output)
        auto count_blocks = [&](const std::vector<OpRec> &ops, const std::vector<char> *starts) {
            int blocks = 0;
            bool pend = false;
            uint32_t c2 = 0, d2 = 0;
            for (size_t oi = 0; oi < ops.size(); ++oi) {
                const OpRec &op = ops[oi];
                if (starts && (*starts)[oi] && pend) { ++blocks; pend = false; c2 = d2 = 0; }
                const uint32_t su = supp(op);
                if (is_perm(op.type)) {
                    if (!pend) continue;
                    if (!(su & d2) && ((su & ~c2) == 0 ||
                                       (starts && __builtin_popcount(c2 | su) <= kBlockBits))) {
                        c2 |= su;
                    } else {
                        d2 |= su;
                    }
                    continue;
                }
                const uint32_t r2 = req(op);
                if ((su & d2) && pend) { ++blocks; pend = false; c2 = d2 = 0; }
                if (op.type == OP_ROTG && __builtin_popcount(op.f) > kBlockBits) {
                    if (pend) ++blocks;
                    ++blocks;
                    pend = false;
                    c2 = d2 = 0;
                    continue;
                }
                if (pend && __builtin_popcount(c2 | r2) > kBlockBits) { ++blocks; pend = false; c2 = d2 = 0; }
                pend = true;
                c2 |= r2;
            }
            return blocks + (pend ? 1 : 0);
        };
        int best = count_blocks(src, nullptr);
        for (int shift = 0; shift < kBlockBits; ++shift) {
            build_order(shift, cand, cand_starts);
            const int nb = count_blocks(cand, &cand_starts);
            if (nb < best) {
                best = nb;
                order.swap(cand);
                cluster_start.swap(cand_starts);
            }
        }
        if (!order.empty()) src.swap(order);
        else cluster_start.clear();
    }
    // Permutations inside an open block whose bits fit the block become
    // register relabelings (free in specialised passes) instead of being
    // deferred to the SMEM map, which would force a new block as soon as a
    // later op touches their qubits (every brickwork CNOT would split blocks).
    const char *env_inreg = getenv("QSV_INREG_PERMS");
    const bool inreg_perms = !(env_inreg && env_inreg[0] == '0');
    for (size_t oi = 0; oi < src.size(); ++oi) {
        const OpRec &op = src[oi];
        if (!cluster_start.empty() && cluster_start[oi] && !pending.empty()) flush();
        if (is_perm(op.type)) {
            if (pending.empty()) {
                apply_perm(op);  // free: only the map changes
            } else if (inreg_perms && !(supp(op) & D) &&
                       ((supp(op) & ~cur) == 0 ||
                        (!cluster_start.empty() && __builtin_popcount(cur | supp(op)) <= kBlockBits))) {
                cur |= supp(op);
                pending.push_back(op);
            } else {
                perms.push_back(op);
                D |= supp(op);
            }
            continue;
        }
        const uint32_t s = supp(op), r = req(op);
        if (s & D) flush();
        if (op.type == OP_ROTG && __builtin_popcount(op.f) > kBlockBits) {
            flush();
            prev_conform = false;
            BlockRec br{};
            br.kind = 1;
            for (int b = 0; b < 12; ++b) br.cols[b] = swz16(A[b]);
            br.tswz = swz16(tr);
            br.op0 = (int)out.size();
            out.push_back(op);
            br.op1 = (int)out.size();
            t.blocks.push_back(br);
            continue;
        }
        if (!pending.empty() && __builtin_popcount(cur | r) > kBlockBits) flush();
        if (pending.empty()) start_block();
        cur |= r;
        pending.push_back(op);
    }
    flush();
    pp.block_end = (int)t.blocks.size();
    for (int b = pp.block_begin; b < pp.block_end; ++b) {
        t.blocks[b].op0 += pp.op_begin;
        t.blocks[b].op1 += pp.op_begin;
    }
    // the pass's ops are the tail of t.ops; a split rotation group can make
    // the block-encoded list longer than the source
    t.ops.erase(t.ops.begin() + pp.op_begin, t.ops.begin() + pp.op_end);
    t.ops.insert(t.ops.begin() + pp.op_begin, out.begin(), out.end());
    pp.op_end = pp.op_begin + (int)out.size();
    pp.map_permuted = tr != 0;
    for (int b = 0; b < 12; ++b) {
        pp.store_cols[b] = swz16(A[b]);
        if (b < m && A[b] != (1u << b)) pp.map_permuted = true;
    }
    pp.store_t = swz16(tr);
    t.n_blocks += pp.block_end - pp.block_begin;
}

}  // namespace

thread_local bool t_plain_u3 = false;
void set_plain_u3(bool on) { t_plain_u3 = on; }
bool plain_u3() { return t_plain_u3; }

bool needs_plain_u3(const ProgramTemplate &t, const double *values)
{
    for (size_t f = 0; f < t.fill_mode.size(); ++f)
        if (t.fill_mode[f] && std::fabs(std::cos(0.5 * values[3 * (size_t)t.fills[f].src])) < 1e-3)
            return true;
    return false;
}


int gate_matrix(int kind, const double *v, double *o)
{
    // circuit.py:36-45 (fixed), :164-171 (_u3_matrix), :198-223 (gate_matrix)
    const double r = std::sqrt(0.5);
    auto set = [&](int i, double re, double im) {
        o[2 * i] = re;
        o[2 * i + 1] = im;
    };
    switch (kind) {
        case K_H: set(0, r, 0); set(1, r, 0); set(2, r, 0); set(3, -r, 0); return 8;
        case K_HY: set(0, r, 0); set(1, 0, -r); set(2, 0, r); set(3, -r, 0); return 8;
        case K_RZ: {
            const double c = std::cos(0.5 * v[0]), s = std::sin(0.5 * v[0]);
            set(0, c, -s);
            set(1, c, s);
            return 4;
        }
        case K_RY: {
            const double c = std::cos(v[0] / 2), s = std::sin(v[0] / 2);
            set(0, c, 0); set(1, -s, 0); set(2, s, 0); set(3, c, 0);
            return 8;
        }
        case K_U3:
        case K_CU3: {
            const double th = v[0], ph = v[1], la = v[2];
            const double c = std::cos(th / 2), s = std::sin(th / 2);
            double u[8];
            u[0] = c; u[1] = 0;
            u[2] = -std::cos(la) * s; u[3] = -std::sin(la) * s;
            u[4] = std::cos(ph) * s; u[5] = std::sin(ph) * s;
            u[6] = std::cos(ph + la) * c; u[7] = std::sin(ph + la) * c;
            if (kind == K_U3) {
                std::memcpy(o, u, sizeof(u));
                return 8;
            }
            for (int i = 0; i < 32; ++i) o[i] = 0.0;
            o[0] = 1.0;            // (0,0)
            o[2 * 5] = 1.0;        // (1,1)
            o[2 * 10] = u[0]; o[2 * 10 + 1] = u[1];   // (2,2)
            o[2 * 11] = u[2]; o[2 * 11 + 1] = u[3];   // (2,3)
            o[2 * 14] = u[4]; o[2 * 14 + 1] = u[5];   // (3,2)
            o[2 * 15] = u[6]; o[2 * 15 + 1] = u[7];   // (3,3)
            return 32;
        }
        default: return 0;
    }
}

TileDims dims_of(const TileGeom &g)
{
    TileDims d;
    d.n = g.n;
    d.m = g.m;
    d.c = g.c;
    d.ncomp = g.ncomp;
    return d;
}

void geom_tables(const TileGeom &g, std::vector<uint64_t> &offhi, std::vector<int32_t> &comp32,
                 const PassPlan *pp)
{
    const int nhi = 1 << (g.m - g.c);
    offhi.assign(nhi, 0);
    for (int i = 0; i < nhi; ++i) {
        uint64_t off = 0;
        for (int b = 0; b < g.m - g.c; ++b)
            if ((i >> b) & 1) off |= 1ull << g.pos[g.c + b];
        offhi[i] = off;
    }
    comp32.assign(64, 0);
    for (int i = 0; i < g.ncomp && i < 32; ++i) comp32[i] = g.comp[i];
    for (int b = 0; b < 12; ++b) {
        const uint32_t l = 1u << b;
        comp32[32 + b] = pp ? pp->store_cols[b] : (int32_t)tile_swz(l);
    }
    comp32[44] = pp ? pp->store_t : 0;
}

void match_rotations(int64_t N, const int32_t *kinds, const int32_t *qubits, std::vector<RotSpan> &out)
{
    out.clear();
    int64_t i = 0;
    while (i < N) {
        Rot rot;
        int64_t len = 0;
        if (match_block(kinds, qubits, N, i, rot, len)) {
            out.push_back(RotSpan{i, len, rot.x, rot.y, rot.z, (int64_t)rot.src});
            i += len;
        } else {
            ++i;
        }
    }
}

// Cache key of a gate structure.  Only a screen: a cache hit is confirmed by
// comparing the full kind / qubit arrays, so the key samples at most 1024
// gates (evenly spaced) and stays O(1) for long UCC circuits.
uint64_t hash_structure(int n_qubits, int64_t n_gates, const int32_t *kinds, const int32_t *qubits)
{
    uint64_t h = 1469598103934665603ull ^ (uint64_t)n_qubits;
    auto mix = [&](uint64_t v) {
        h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
        h *= 1099511628211ull;
    };
    mix((uint64_t)n_gates);
    const int64_t step = n_gates > 1024 ? n_gates / 1024 : 1;
    for (int64_t i = 0; i < n_gates; i += step) {
        mix(((uint64_t)(uint32_t)kinds[i] << 40) ^ ((uint64_t)(uint32_t)qubits[2 * i] << 20) ^
            (uint64_t)(uint32_t)qubits[2 * i + 1]);
    }
    return h;
}

// QSV_SCHED: "order" (first fit in circuit order, backfilling earlier passes),
// "lookahead" (above); default: both, keep the one with fewer passes.
Schedule pick_schedule(const std::vector<Item> &items, const std::vector<Rot> &R, int n, int m, int c)
{
    const char *env = getenv("QSV_SCHED");
    const char *env_cap = getenv("QSV_PASS_COST_CAP");
    const int cost_cap = env_cap ? std::max(1, atoi(env_cap)) : 128;
    if (env && std::string(env) == "order") return schedule(items, R, n, m, c);
    if (items.size() > 20000) return schedule(items, R, n, m, c);  // O(N^2) conflict graph
    const char *env_win = getenv("QSV_SCHED_WINDOW");
    const int window = env_win ? std::max(8, atoi(env_win)) : 512;
    Schedule L = schedule_lookahead(items, R, m, c, cost_cap, window);
    if (env && std::string(env) == "lookahead") return L;
    Schedule O = schedule(items, R, n, m, c);
    return L.pass_items.size() < O.pass_items.size() ? L : O;
}

// Rotation-dominated (UCC) programs on specialised tiles are bound by HBM and by
// tile capacity: 2 contiguous low qubits (64-B segments) leave 10 tile slots
// for flip bits instead of 9, so fewer passes, at a lower per-pass HBM
// efficiency.  Measured on B200 (30 q UCC, 16,450 rotations): c = 3: 691
// passes at 0.83 of peak (4.37 s); c = 2: 621 passes at 0.78 (4.16 s).  Keep
// the schedule with the smaller passes / efficiency (QSV_MIN_CONTIG pins c).
void pick_contig(const std::vector<Item> &items, const std::vector<Rot> &R, int n, int m, int &c,
                 Schedule &S)
{
    if (getenv("QSV_MIN_CONTIG") || n < 22 || m != kMaxTileBits || c != 3) return;
    size_t nrot = 0;
    for (const Item &it : items) nrot += it.rot ? 1 : 0;
    if (nrot * 2 < items.size()) return;  // gate circuits: FP64-bound, c = 3 measured best
    Schedule S2 = pick_schedule(items, R, n, m, 2);
    if ((double)S2.pass_items.size() / 0.78 < (double)S.pass_items.size() / 0.83) {
        S = std::move(S2);
        c = 2;
    }
}

void plan_gates(int n, int64_t N, const int32_t *kinds, const int32_t *qubits, ProgramTemplate &t)
{
    t = ProgramTemplate();
    int m, c;
    choose_tile(n, m, c);
    std::vector<Rot> R;
    std::vector<Item> items;
    int64_t i = 0;
    bool all_rot = true;
    while (i < N) {
        Rot rot;
        int64_t len = 0;
        if (match_block(kinds, qubits, N, i, rot, len)) {
            const uint64_t a = rot.x | rot.y, b = rot.y | rot.z;
            R.push_back(rot);
            const int r = (int)R.size() - 1;
            if (!items.empty() && items.back().rot && items.back().req == a) {
                Item &g = items.back();
                g.rots.push_back(r);
                g.b_union |= b;
                g.supp |= a | b;
                if (rot.z != g.last_z) g.par += rot_par(a);  // a run of another sign mask: its own table
                g.last_z = rot.z;
            } else {
                Item it;
                it.rot = true;
                it.cost = 0;  // a same-flip group is one GMAT per sign-mask run: bounded by the parameter budget
                it.par = rot_par(a);
                it.last_z = rot.z;
                it.rots.push_back(r);
                it.a_union = a;
                it.b_union = b;
                it.supp = a | b;
                it.req = a;
                items.push_back(std::move(it));
            }
            i += len;
        } else {
            all_rot = false;
            Item it;
            it.gate = (int)i;
            uint64_t s = 1ull << qubits[2 * i];
            if (qubits[2 * i + 1] >= 0) s |= 1ull << qubits[2 * i + 1];
            it.supp = s;
            it.req = s;
            it.cost = gate_cost(kinds[i]);
            it.par = gate_par(kinds[i]);
            items.push_back(std::move(it));
            ++i;
        }
    }
    fuse_clusters(items, kinds, qubits, t);
    find_phase_defers(items, kinds, qubits, n, t);
    find_cz_defers(items, kinds, qubits, n, m, t);
    Schedule S = pick_schedule(items, R, n, m, c);
    pick_contig(items, R, n, m, c, S);
    emit_program(n, m, c, items, R, kinds, qubits, S, t);
    t.n_input = N;
    t.src_kinds.assign(kinds, kinds + N);
    t.src_qubits.assign(qubits, qubits + 2 * N);
    t.n_rotations = (int64_t)R.size();
    if (all_rot && n <= kSmallMaxQubits) build_small_program(n, R, t.small);
}

void plan_rotations(int n, const std::vector<Rot> &R, int64_t n_input, ProgramTemplate &t)
{
    t = ProgramTemplate();
    int m, c;
    choose_tile(n, m, c);
    std::vector<Item> items;
    build_items_from_rots(R, items);
    Schedule S = pick_schedule(items, R, n, m, c);
    pick_contig(items, R, n, m, c, S);
    emit_program(n, m, c, items, R, nullptr, nullptr, S, t);
    t.n_input = n_input;
    t.n_rotations = (int64_t)R.size();
}

void materialize_gates(ProgramTemplate &t, const double *values)
{
    for (size_t r = 0; r < t.rots.size(); ++r) {
        const double th = values[3 * (size_t)t.rot_src[r]];
        t.rots[r].c = std::cos(0.5 * th);
        t.rots[r].s = std::sin(0.5 * th);
    }
}

void materialize_params(ProgramTemplate &t, const double *values, double *params, bool with_gmats)
{
    materialize_gates(t, values);
    const bool norm = !t.fill_mode.empty() && !t.pass_sink.empty();
    if (t.defers.empty() && t.czdefers.empty() && !norm) {
        for (const ParamFill &f : t.fills) gate_matrix(f.kind, values + 3 * (size_t)f.src, params + f.offset);
    } else {
        // deferred phases: a deferring U3 hands phi (and, in shear mode, its
        // effective lambda) to its receiving U3; processed in gate order so
        // chains of deferrals accumulate
        std::unordered_map<int, int8_t> mode_of;  // gate -> fill mode
        if (norm)
            for (size_t f = 0; f < t.fills.size(); ++f)
                if (f < t.fill_mode.size() && t.fill_mode[f]) mode_of[t.fills[f].src] = t.fill_mode[f];
        // both deferral kinds, in source gate order (a source's effective
        // lambda includes what earlier sources handed it)
        struct Dv { int src, dst, ctl; };
        std::vector<Dv> ds;
        for (const PhaseDefer &d : t.defers) ds.push_back({d.src, d.dst, -1});
        for (const CzDefer &d : t.czdefers) ds.push_back({d.src, d.tgt, d.ctl});
        std::sort(ds.begin(), ds.end(), [](const Dv &a, const Dv &b) { return a.src < b.src; });
        std::unordered_map<int, double> add_lambda;  // receiving gate -> deferred phase
        std::unordered_map<int, double> ctl_lambda;  // OP_U1C gate -> extra lambda when its control is 1
        std::unordered_map<int, char> deferring;
        for (const Dv &d : ds) {
            deferring[d.src] = 1;
            double give = values[3 * (size_t)d.src + 1];  // phi
            auto m = mode_of.find(d.src);
            if (m != mode_of.end() && m->second == 6) {
                auto a = add_lambda.find(d.src);
                give += values[3 * (size_t)d.src + 2] + (a != add_lambda.end() ? a->second : 0.0);
            }
            add_lambda[d.dst] += give;
            if (d.ctl >= 0) {  // e^{ib (x_t ^ x_c)} = e^{ib x_t} e^{ib x_c} e^{-2ib x_t x_c}
                add_lambda[d.ctl] += give;
                ctl_lambda[d.ctl] -= 2.0 * give;
            }
        }
        std::vector<double> mu(t.pass_sink.size(), 1.0);
        for (size_t fi = 0; fi < t.fills.size(); ++fi) {
            const ParamFill &f = t.fills[fi];
            const double *v = values + 3 * (size_t)f.src;
            if (f.kind != K_U3) {
                gate_matrix(f.kind, v, params + f.offset);
                continue;
            }
            double vv[3] = {v[0], v[1], v[2]};
            auto it = add_lambda.find(f.src);
            if (it != add_lambda.end()) vv[2] += it->second;
            if (deferring.count(f.src)) vv[1] = 0.0;  // V = U3(t, 0, l): the phi phase moves on
            const int mode = norm && fi < t.fill_mode.size() ? t.fill_mode[fi] : 0;
            double *o = params + f.offset;
            if (mode == 6) {  // c diag(1, e^{il}) [[1, -e^{il} tn], [e^{-il} tn, 1]]
                const double c = std::cos(0.5 * vv[0]), tn = std::tan(0.5 * vv[0]);
                const double cl = std::cos(vv[2]), sl = std::sin(vv[2]);
                o[0] = 1.0; o[1] = 0.0;
                o[2] = -cl * tn; o[3] = -sl * tn;
                o[4] = cl * tn; o[5] = -sl * tn;
                o[6] = 1.0; o[7] = 0.0;
                mu[t.fill_pass[fi]] *= c;
                continue;
            }
            gate_matrix(K_U3, vv, o);
            if (f.ctrl) {  // OP_U1C: the matrix for control bit 1 follows
                double v1[3] = {vv[0], vv[1], vv[2]};
                auto cl = ctl_lambda.find(f.src);
                if (cl != ctl_lambda.end()) v1[2] += cl->second;
                gate_matrix(K_U3, v1, o + 8);
            }
            if (mode == 4) {  // U3 / c: m00 = 1 exactly (both matrices of an OP_U1C)
                const double c = o[0], inv = 1.0 / c;
                for (int h = 0; h <= f.ctrl; ++h) {
                    double *q = o + 8 * h;
                    for (int k = 2; k < 8; ++k) q[k] *= inv;
                    q[0] = 1.0;
                    q[1] = 0.0;
                }
                mu[t.fill_pass[fi]] *= c;
            }
        }
        if (norm)
            for (size_t p = 0; p < t.pass_sink.size(); ++p)
                if (t.pass_sink[p] >= 0 && mu[p] != 1.0) {
                    const ParamFill &sf = t.fills[t.pass_sink[p]];
                    double *o = params + sf.offset;
                    for (int k = 0; k < 8 * (1 + sf.ctrl); ++k) o[k] *= mu[p];
                }
    }
    for (const ClusterFill &cf : t.cfills)
        if (cf.offset >= 0)
            cluster_matrix(cf, t.src_kinds.data(), t.src_qubits.data(), values, params + cf.offset);
    if (with_gmats) materialize_gmats(t, params);
}

void materialize_rotations(ProgramTemplate &t, const double *theta)
{
    for (size_t r = 0; r < t.rots.size(); ++r) {
        const double th = theta[t.rot_src[r]];
        t.rots[r].c = std::cos(0.5 * th);
        t.rots[r].s = std::sin(0.5 * th);
    }
}

void materialize_gmats(const ProgramTemplate &t, double *params)
{
    static const std::vector<uint8_t> par8 = [] {
        std::vector<uint8_t> v(256);
        for (int i = 0; i < 256; ++i) v[i] = (uint8_t)(__builtin_popcount((unsigned)i) & 1);
        return v;
    }();
    std::vector<double> kre, kim;
    std::vector<uint8_t> yodd;
    for (const GmatFill &g : t.gfills) {
        const int ncfg = 1 << (g.w - 1);
        const int nr = g.r1 - g.r0;
        // kappa = i^q sin per rotation; R = [[c, kappa sg1], [kappa sg0, c]]
        kre.assign(nr, 0.0);
        kim.assign(nr, 0.0);
        yodd.resize(nr);
        for (int r = 0; r < nr; ++r) {
            const RotRec &R = t.rots[g.r0 + r];
            yodd[r] = (uint8_t)((R.q >> 2) & 1);
            switch (R.q & 3) {
                case 0: kre[r] = R.s; break;
                case 1: kim[r] = R.s; break;
                case 2: kre[r] = -R.s; break;
                default: kim[r] = -R.s; break;
            }
        }
        int fpos[8], k = 0;
        for (int j = 0; j < 8; ++j)
            if ((g.F >> j) & 1) fpos[k++] = j;
        for (int cfg = 0; cfg < ncfg; ++cfg) {
            // r1's bits on F: bit H set, the others from cfg (ascending, H skipped)
            uint32_t r1 = 1u << g.H;
            for (int i = 0, c = 0; i < g.w; ++i) {
                if (fpos[i] == g.H) continue;
                if ((cfg >> c) & 1) r1 |= 1u << fpos[i];
                ++c;
            }
            double M[8] = {1, 0, 0, 0, 0, 0, 1, 0};  // identity, row-major complex
            for (int r = 0; r < nr; ++r) {
                const double cr = t.rots[g.r0 + r].c;
                const int s1 = par8[(r1 & g.yF[r]) & 255u];
                const int s0 = s1 ^ yodd[r];
                const double b_re = s1 ? -kre[r] : kre[r], b_im = s1 ? -kim[r] : kim[r];
                const double c_re = s0 ? -kre[r] : kre[r], c_im = s0 ? -kim[r] : kim[r];
                // M <- R M with R = [[c, b], [cc, c]]: rows mix, two columns
                for (int j = 0; j < 2; ++j) {
                    const double a0r = M[2 * j], a0i = M[2 * j + 1];
                    const double a1r = M[4 + 2 * j], a1i = M[4 + 2 * j + 1];
                    M[2 * j] = cr * a0r + (b_re * a1r - b_im * a1i);
                    M[2 * j + 1] = cr * a0i + (b_re * a1i + b_im * a1r);
                    M[4 + 2 * j] = cr * a1r + (c_re * a0r - c_im * a0i);
                    M[4 + 2 * j + 1] = cr * a1i + (c_re * a0i + c_im * a0r);
                }
            }
            // common parity cp = 1 negates every off-diagonal factor:
            // R' = Z R Z, so the product is Z M Z (exactly: only signs change)
            double *d0 = params + g.offset + 8 * cfg;
            double *d1 = params + g.offset + 8 * (ncfg + cfg);
            for (int i = 0; i < 8; ++i) d0[i] = M[i];
            d1[0] = M[0];
            d1[1] = M[1];
            d1[2] = -M[2];
            d1[3] = -M[3];
            d1[4] = -M[4];
            d1[5] = -M[5];
            d1[6] = M[6];
            d1[7] = M[7];
        }
    }
}

// ---------------------------------------------------------------------------
// Expectation sweeps
// ---------------------------------------------------------------------------

// Reorder terms [a, b) so that consecutive terms read different shared-memory
// banks in the tile-wide transform lookups (index wpos(s) = s ^ ((s >> 4) & 15)
// within a 2048-double half: bank pair = its low 4 bits): round-robin over the
// 16 bank buckets, so a half-warp's 16 lookups are conflict-free when the
// buckets are balanced.  Term order inside a sweep is free (map[] restores it).
void bank_interleave(std::vector<TermRec> &terms, std::vector<int32_t> &map, size_t a, size_t b)
{
    if (b - a < 2) return;
    std::vector<std::vector<size_t>> bucket(16);
    for (size_t i = a; i < b; ++i) {
        const uint32_t sp = terms[i].s_loc & 2047u;
        bucket[(sp ^ (sp >> 4)) & 15u].push_back(i);
    }
    std::vector<TermRec> t2;
    std::vector<int32_t> m2;
    t2.reserve(b - a);
    m2.reserve(b - a);
    for (size_t round = 0; t2.size() < b - a; ++round)
        for (int k = 0; k < 16; ++k)
            if (round < bucket[k].size()) {
                t2.push_back(terms[bucket[k][round]]);
                m2.push_back(map[bucket[k][round]]);
            }
    std::copy(t2.begin(), t2.end(), terms.begin() + a);
    std::copy(m2.begin(), m2.end(), map.begin() + a);
}

void plan_expectation(int n, int64_t S, const uint64_t *x, const uint64_t *y, const uint64_t *z,
                      std::vector<SweepPlan> &out, bool jit_layout)
{
    out.clear();
    int m, c;
    choose_tile(n, m, c);
    const uint64_t low = c >= 64 ? ~0ull : ((1ull << c) - 1ull);
    const int free_slots = m - c;
    const int kCap = 2048;  // terms per sweep (shared-memory accumulators)

    std::vector<int32_t> diag;
    std::unordered_map<uint64_t, int> flip_index;
    std::vector<uint64_t> flips;
    std::vector<std::vector<int32_t>> members;
    for (int64_t t = 0; t < S; ++t) {
        const uint64_t f = x[t] | y[t];
        if (f == 0) {
            diag.push_back((int32_t)t);
            continue;
        }
        auto it = flip_index.find(f);
        if (it == flip_index.end()) {
            flip_index.emplace(f, (int)flips.size());
            flips.push_back(f);
            members.emplace_back();
            members.back().push_back((int32_t)t);
        } else {
            members[it->second].push_back((int32_t)t);
        }
    }
    // Bin flip groups into sweeps: a sweep's tile must hold every group's
    // flip bits.  First-fit decreasing on the high-bit need; capacity is
    // bounded by the shared-memory accumulators (kFlipCap strings).
    const char *env_sc = getenv("QSV_SWEEP_TERMS");  // strings per specialised sweep (default 24)
    const int jit_cap = env_sc ? std::max(4, std::min(48, atoi(env_sc))) : 24;
    // per-warp specialised sweeps (QSV_SWEEP_WARPS=1, qsv_jit.cpp
    // jit_sweep_source_warps): each of the 8 warps of a tile group holds <=
    // jit_cap strings -- half the sweeps on config 3, but measured 1.4 s vs
    // 0.8 s (profiles/r02_expect30_warps_launches.csv), so off by default
    const char *env_w = getenv("QSV_SWEEP_WARPS");
    const int warps = jit_layout && env_w && env_w[0] == '1' ? 8 : 1;
    const int kFlipCap = jit_layout ? jit_cap * warps : 512, kDiagCap = 2048, kGroupCap = 256;
    std::vector<int> order(flips.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        if (jit_layout) {
            // specialised sweeps share the l0-side loads of groups with the
            // same highest flip bit: keep such groups adjacent
            const int ha = highest_bit(flips[a]), hb = highest_bit(flips[b]);
            if (ha != hb) return ha > hb;
        }
        const int pa = popc64(flips[a] & ~low), pb = popc64(flips[b] & ~low);
        if (pa != pb) return pa > pb;
        return members[a].size() > members[b].size();
    });
    struct Bin {
        uint64_t hi = 0;
        int nterms = 0;
        int wl[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // strings per warp (per-warp sweeps)
        bool wide = false;
        std::vector<int> groups;
        std::vector<int32_t> diag;
    };
    // Wide groups (more strings than a specialised sweep holds) take the
    // tile-wide Walsh-Hadamard path of the interpreted sweep: one transform of
    // the group's pair products per tile, then one lookup per string -- so
    // they share sweeps (with the Z-only strings) instead of one sweep each.
    const int kWideMin = jit_layout ? jit_cap : 24, kWideCap = 2048;
    const bool wide_ok = m == kMaxTileBits;
    std::vector<Bin> bins;
    std::vector<int> global_groups;
    for (int gi : order) {
        const uint64_t need = flips[gi] & ~low;
        const int nt = (int)members[gi].size();
        const bool wide = wide_ok && nt > kWideMin;
        if (popc64(need) > free_slots || nt > (wide ? kWideCap : 512)) {
            global_groups.push_back(gi);
            continue;
        }
        const int cap = wide ? kWideCap : kFlipCap;
        int placed = -1;
        // a narrow group above the (specialised-sweep) cap gets a sweep of its own
        auto warp_of = [&](const Bin &bn) {  // a warp with room for nt more strings, -1 if none
            if (wide || warps == 1) return 0;
            for (int w = 0; w < warps; ++w)
                if (bn.wl[w] + nt <= jit_cap) return w;
            return -1;
        };
        for (size_t b = 0; b < bins.size() && nt <= cap; ++b) {
            if (bins[b].wide != wide) continue;
            if (bins[b].nterms + nt > cap || (int)bins[b].groups.size() >= kGroupCap) continue;
            if (warp_of(bins[b]) < 0) continue;
            if (popc64(bins[b].hi | need) <= free_slots) {
                placed = (int)b;
                break;
            }
        }
        if (placed < 0) {
            bins.emplace_back();
            bins.back().wide = wide;
            placed = (int)bins.size() - 1;
        }
        {
            const int w = warp_of(bins[placed]);
            if (w >= 0) bins[placed].wl[w] += nt;
        }
        bins[placed].hi |= need;
        bins[placed].nterms += nt;
        bins[placed].groups.push_back(gi);
    }
    // Z-only strings ride along with the wide sweeps, else the first sweeps
    // (any tile works), or -- for the specialised flip-only kernel -- sweeps
    // of their own
    std::vector<size_t> diag_bins;
    for (size_t b = 0; b < bins.size(); ++b)
        if (bins[b].wide) diag_bins.push_back(b);
    if (!jit_layout)
        for (size_t b = 0; b < bins.size(); ++b)
            if (!bins[b].wide) diag_bins.push_back(b);
    for (size_t d0 = 0, k = 0; d0 < diag.size(); d0 += kDiagCap, ++k) {
        if (k >= diag_bins.size()) {
            bins.emplace_back();
            diag_bins.push_back(bins.size() - 1);
        }
        bins[diag_bins[k]].diag.assign(diag.begin() + d0,
                                       diag.begin() + std::min(diag.size(), d0 + kDiagCap));
    }

    auto term_scale = [&](int64_t t) {
        const int ny = popc64(y[t]);
        if ((ny & 1) == 0) return ((ny / 2) & 1) ? -2.0 : 2.0;
        return (((ny + 1) / 2) & 1) ? 2.0 : -2.0;
    };

    for (Bin &bin : bins) {
        SweepPlan sp;
        sp.geom = make_geom(n, m, c, bin.hi);
        const uint64_t tm = tile_mask(sp.geom);
        sp.ndiag = (int)bin.diag.size();
        for (int32_t t : bin.diag) {
            TermRec tr{};
            const uint64_t bb = y[t] | z[t];
            tr.s_hi = bb & ~tm;
            tr.s_loc = compress(bb, sp.geom);
            tr.use_im = 0;
            tr.scale = 1.0;
            sp.terms.push_back(tr);
            sp.map.push_back(t);
        }
        if (m == kMaxTileBits) bank_interleave(sp.terms, sp.map, 0, sp.terms.size());
        // heavier groups first so the two warp halves stay balanced; with the
        // specialised layout, groups with the same highest flip bit adjacent
        // specialised sweeps: within a run, flips that differ only in the
        // tile positions of pair bits 8..10 adjacent (they share one load of
        // the l1-side amplitudes, jit_sweep_source)
        auto share_key = [&](int g) {
            const uint32_t fl = compress(flips[g], sp.geom);
            const int H = highest_bit(fl);
            uint32_t R = 0;
            for (int k = 0; k < 3; ++k) R |= 1u << ((8 + k) + ((8 + k) >= H ? 1 : 0));
            return fl & ~R;
        };
        std::stable_sort(bin.groups.begin(), bin.groups.end(), [&](int a, int b) {
            if (jit_layout) {
                const int ha = highest_bit(flips[a]), hb = highest_bit(flips[b]);
                if (ha != hb) return ha > hb;
                const uint32_t ka = share_key(a), kb = share_key(b);
                if (ka != kb) return ka < kb;
            }
            return members[a].size() > members[b].size();
        });
        for (int gi : bin.groups) {
            GroupRec gr{};
            gr.f_loc = compress(flips[gi], sp.geom);
            gr.h = highest_bit(gr.f_loc);
            gr.pad[0] = bin.wide ? 1 : 0;  // tile-wide transform path
            const uint32_t lowmask_h = (1u << gr.h) - 1u;
            gr.t0 = (int)sp.terms.size();
            for (int pass = 0; pass < 2; ++pass) {  // Re-w strings, then Im-w strings
                if (pass == 1) gr.t_im = (int)sp.terms.size();
                for (int32_t t : members[gi]) {
                    if ((popc64(y[t]) & 1) != pass) continue;
                    TermRec tr{};
                    const uint64_t bb = y[t] | z[t];
                    const uint32_t sl = compress(bb, sp.geom);
                    tr.s_hi = bb & ~tm;
                    // sign mask in pair-index coordinates (bit h removed)
                    tr.s_loc = (sl & lowmask_h) | ((sl >> (gr.h + 1)) << gr.h);
                    tr.use_im = pass;
                    tr.scale = term_scale(t);
                    sp.terms.push_back(tr);
                    sp.map.push_back(t);
                }
            }
            gr.t1 = (int)sp.terms.size();
            if (bin.wide) {  // tile-wide path: one lookup per string per tile
                bank_interleave(sp.terms, sp.map, gr.t0, gr.t_im);
                bank_interleave(sp.terms, sp.map, gr.t_im, gr.t1);
            }
            sp.groups.push_back(gr);
        }
        out.push_back(std::move(sp));
    }
    // global fallback sweeps (flip too wide for a tile): chunks of groups
    size_t gpos = 0;
    while (gpos < global_groups.size()) {
        SweepPlan sp;
        sp.global = true;
        std::memset(&sp.geom, 0, sizeof(sp.geom));
        sp.geom.n = n;
        while (gpos < global_groups.size() &&
               (int)sp.terms.size() + (int)members[global_groups[gpos]].size() <= kCap) {
            const int gi = global_groups[gpos++];
            GroupRec gr{};
            gr.f_loc = 0;
            gr.h = highest_bit(flips[gi]);
            gr.t0 = (int)sp.terms.size();
            for (int32_t t : members[gi]) {
                TermRec tr{};
                tr.s_hi = y[t] | z[t];
                tr.s_loc = 0;
                tr.use_im = popc64(y[t]) & 1;
                tr.scale = term_scale(t);
                sp.terms.push_back(tr);
                sp.map.push_back(t);
            }
            gr.t1 = (int)sp.terms.size();
            sp.groups.push_back(gr);
            sp.gflip.push_back(flips[gi]);
        }
        if (sp.groups.empty()) {  // a single group larger than the cap: split its terms
            const int gi = global_groups[gpos++];
            const auto &mem = members[gi];
            for (size_t k0 = 0; k0 < mem.size(); k0 += kCap) {
                SweepPlan s2;
                s2.global = true;
                std::memset(&s2.geom, 0, sizeof(s2.geom));
                s2.geom.n = n;
                GroupRec gr{};
                gr.h = highest_bit(flips[gi]);
                gr.t0 = 0;
                for (size_t k = k0; k < std::min(mem.size(), k0 + kCap); ++k) {
                    const int32_t t = mem[k];
                    TermRec tr{};
                    tr.s_hi = y[t] | z[t];
                    tr.use_im = popc64(y[t]) & 1;
                    tr.scale = term_scale(t);
                    s2.terms.push_back(tr);
                    s2.map.push_back(t);
                }
                gr.t1 = (int)s2.terms.size();
                s2.groups.push_back(gr);
                s2.gflip.push_back(flips[gi]);
                out.push_back(std::move(s2));
            }
            continue;
        }
        out.push_back(std::move(sp));
    }
}

}  // namespace qsv
