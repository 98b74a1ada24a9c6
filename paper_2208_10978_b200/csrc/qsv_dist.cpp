// qsv_dist.cpp -- native multi-device state (one process driving P shards).
//
// The C-ABI counterpart of distributed.py for callers that drive several GPUs
// from one process (qsv_create(.., n_devices, device_ids);
// the reference's own parallel model is one process forking workers,
// engine.py:169-199).  The layout, planner and reduction order are those of
// distributed.py: rank r holds the 2^(n-g) amplitudes whose physical index
// bits [n_local, n) equal r; a logical -> physical qubit map is tracked and
// never swapped back; a gate list is cut into local segments by the
// local-first light-cone scheduler (plan_segments) with qubit-swap relayouts
// between them; expectation values are reduced over ranks in ascending order
// (engine.py:199).  Shards are ordinary qsv_state handles, so every local pass
// is the single-GPU engine.  A relayout swaps contiguous chunks pairwise IN
// PLACE over peer memory: a swap kernel reads and writes both chunks directly
// (NVLink / NVSwitch P2P loads and stores; plain device memory when two ranks
// share a device), each device of a pair swapping one half, ordered against
// the shards' other work by events -- no staging copy, no host round trip.
// Without peer access (or QSV_DIST_P2P=0) the swap falls back to
// cudaMemcpyPeerAsync through a bounded staging piece.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "../../include/qsv.h"
#include "qsv_internal.h"
#include "qsv_planner.h"

struct qsv_dist {
    int n = 0, n_local = 0, g = 0, P = 0;
    std::vector<int> devices;         // per rank
    std::vector<qsv_state *> shards;  // per rank
    std::vector<int> perm;            // logical qubit -> physical position
    std::vector<void *> staging;      // per rank: one piece on the rank's device
    size_t piece_bytes = 64u << 20;
    bool p2p = false;                 // every pair of devices can address each other
    std::vector<cudaEvent_t> ev_ready, ev_done;  // per rank: relayout ordering
    int64_t swap_launches = 0;
    bool lazy = false;                // |basis> not yet materialised
    uint64_t basis = 0;
    int64_t relayouts = 0, bytes_sent = 0;  // per rank
};

namespace qsv {
namespace {

std::recursive_mutex d_mu;

int fail_code(int code, const std::string &msg)
{
    set_error(msg);  // the thread's qsv_last_error()
    return code;
}

constexpr int kSwap = 4;  // gate kind code of SWAP (include/qsv.h)

int gate_qubits(const int32_t *qubits, int64_t i, int out[2])
{
    out[0] = qubits[2 * i];
    out[1] = qubits[2 * i + 1];
    return out[1] < 0 ? 1 : 2;
}

struct Relayout {
    std::vector<int> S;  // global bit indices swapped with the top |S| local positions
};

struct Segment {
    std::vector<int64_t> src;    // source gate per local gate, -1: inserted SWAP
    std::vector<int32_t> qubits; // 2 per local gate, physical local positions
    bool has_relayout = false;
    Relayout rl;
};

void move_victims(std::vector<int> &perm, std::vector<int> &inv, const std::vector<int> &victims,
                  int n_local, std::vector<std::pair<int, int>> &swaps)
{
    const int k = (int)victims.size();
    for (int j = 0; j < k; ++j) {
        const int v = victims[j], T = n_local - k + j, p = perm[v];
        if (p != T) {
            const int other = inv[T];
            swaps.push_back({p, T});
            perm[v] = T;
            perm[other] = p;
            inv[T] = v;
            inv[p] = other;
        }
    }
}

void apply_relayout_to_map(std::vector<int> &perm, std::vector<int> &inv, const std::vector<int> &bring,
                           const std::vector<int> &victims, int n_local)
{
    const int k = (int)bring.size();
    for (int j = 0; j < k; ++j) {
        const int b = bring[j], v = victims[j], T = n_local - k + j, G = perm[b];
        perm[b] = T;
        perm[v] = G;
        inv[T] = b;
        inv[G] = v;
    }
}

// distributed.py plan_segments: local-first light-cone scheduling.
bool plan_segments(int64_t N, const int32_t *qubits, int n, int n_local, std::vector<int> &perm,
                   std::vector<Segment> &segs, std::string &err)
{
    const int g = n - n_local;
    std::vector<int> inv(n);
    for (int q = 0; q < n; ++q) inv[perm[q]] = q;
    std::vector<int64_t> remaining(N);
    for (int64_t i = 0; i < N; ++i) remaining[i] = i;
    Segment cur;
    for (;;) {
        std::vector<char> blocked(n, 0);
        std::vector<int64_t> deferred;
        for (int64_t i : remaining) {
            int gq[2];
            const int nq = gate_qubits(qubits, i, gq);
            bool defer = false;
            for (int k = 0; k < nq; ++k) defer |= blocked[gq[k]] || perm[gq[k]] >= n_local;
            if (defer) {
                deferred.push_back(i);
                for (int k = 0; k < nq; ++k) blocked[gq[k]] = 1;
            } else {
                cur.src.push_back(i);
                cur.qubits.push_back(perm[gq[0]]);
                cur.qubits.push_back(nq == 2 ? perm[gq[1]] : -1);
            }
        }
        remaining.swap(deferred);
        if (remaining.empty()) break;
        std::vector<int> bring;
        std::vector<int64_t> first_use(n, INT64_MAX);
        for (size_t pos = 0; pos < remaining.size(); ++pos) {
            int gq[2];
            const int nq = gate_qubits(qubits, remaining[pos], gq);
            for (int k = 0; k < nq; ++k) {
                const int q = gq[k];
                if (first_use[q] == INT64_MAX) first_use[q] = (int64_t)pos;
                if (perm[q] >= n_local && std::find(bring.begin(), bring.end(), q) == bring.end() &&
                    (int)bring.size() < g)
                    bring.push_back(q);
            }
        }
        int head[2];
        const int nh = gate_qubits(qubits, remaining[0], head);
        std::vector<int> cand;
        for (int p = 0; p < n_local; ++p) {
            const int q = inv[p];
            bool skip = std::find(bring.begin(), bring.end(), q) != bring.end();
            for (int k = 0; k < nh; ++k) skip |= head[k] == q;
            if (!skip) cand.push_back(q);
        }
        std::sort(cand.begin(), cand.end(), [&](int a, int b) {
            if (first_use[a] != first_use[b]) return first_use[a] > first_use[b];
            return a < b;
        });
        if (cand.size() < bring.size()) {
            err = "too few local qubits for a relayout";
            return false;
        }
        std::vector<int> victims(cand.begin(), cand.begin() + bring.size());
        std::vector<std::pair<int, int>> swaps;
        move_victims(perm, inv, victims, n_local, swaps);
        for (auto &sw : swaps) {
            cur.src.push_back(-1);
            cur.qubits.push_back(sw.first);
            cur.qubits.push_back(sw.second);
        }
        cur.has_relayout = true;
        cur.rl.S.clear();
        for (int b : bring) cur.rl.S.push_back(perm[b] - n_local);
        segs.push_back(std::move(cur));
        cur = Segment();
        apply_relayout_to_map(perm, inv, bring, victims, n_local);
    }
    segs.push_back(std::move(cur));
    return true;
}

int sync_all(qsv_dist *d)
{
    for (qsv_state *s : d->shards) {
        if (cudaSetDevice(s->device) != cudaSuccess || cudaStreamSynchronize(s->stream) != cudaSuccess)
            return fail_code(QSV_ERR_CUDA, "shard synchronisation failed");
    }
    return QSV_OK;
}

// Swap the top k = |S| local bits with global bits S: rank r exchanges its
// chunk c (c != its own S-pattern) with chunk s(r) of the partner whose
// S-bits are c; chunks are 2^(n_local - k) contiguous amplitudes.
int relayout(qsv_dist *d, const Relayout &rl)
{
    const int k = (int)rl.S.size();
    if (k == 0) return QSV_OK;
    const uint64_t chunk = 1ull << (d->n_local - k);
    auto s_value = [&](int r) {
        int v = 0;
        for (int i = 0; i < k; ++i) v |= ((r >> rl.S[i]) & 1) << i;
        return v;
    };
    auto partner = [&](int r, int c) {
        int p = r;
        for (int i = 0; i < k; ++i) p = (p & ~(1 << rl.S[i])) | (((c >> i) & 1) << rl.S[i]);
        return p;
    };
    const char *knob = getenv("QSV_DIST_P2P");
    if (d->p2p && !(knob && knob[0] == '0')) {
        // every shard's earlier work precedes any swap touching it: rank r's
        // stream waits for the partners' ready events, swaps its half of
        // each pair, and later work on r waits for the partners' done events
        for (int r = 0; r < d->P; ++r) {
            cudaSetDevice(d->devices[r]);
            if (cudaEventRecord(d->ev_ready[r], d->shards[r]->stream) != cudaSuccess)
                return fail_code(QSV_ERR_CUDA, "relayout event record failed");
        }
        for (int r = 0; r < d->P; ++r) {
            qsv_state *A = d->shards[r];
            cudaSetDevice(A->device);
            const int rs = s_value(r);
            for (int c = 0; c < (1 << k); ++c) {
                if (c == rs) continue;
                const int p = partner(r, c);
                if (cudaStreamWaitEvent(A->stream, d->ev_ready[p], 0) != cudaSuccess)
                    return fail_code(QSV_ERR_CUDA, "relayout event wait failed");
            }
            for (int c = 0; c < (1 << k); ++c) {
                if (c == rs) continue;
                const int p = partner(r, c);
                // the pair {r, p}: r's chunk c <-> p's chunk rs; the lower
                // rank swaps the first half, the higher one the second
                const uint64_t half = chunk / 2;
                const uint64_t off = p > r ? 0 : half, len = p > r ? half : chunk - half;
                double2 *a = A->amps + (uint64_t)c * chunk + off;
                double2 *b = d->shards[p]->amps + (uint64_t)rs * chunk + off;
                if (launch_swap_chunks(a, b, len, num_sms(A->device), A->stream) != cudaSuccess)
                    return fail_code(QSV_ERR_CUDA, "relayout swap kernel failed");
                ++d->swap_launches;
            }
            if (cudaEventRecord(d->ev_done[r], A->stream) != cudaSuccess)
                return fail_code(QSV_ERR_CUDA, "relayout event record failed");
        }
        for (int r = 0; r < d->P; ++r) {
            qsv_state *A = d->shards[r];
            cudaSetDevice(A->device);
            const int rs = s_value(r);
            for (int c = 0; c < (1 << k); ++c) {
                if (c == rs) continue;
                if (cudaStreamWaitEvent(A->stream, d->ev_done[partner(r, c)], 0) != cudaSuccess)
                    return fail_code(QSV_ERR_CUDA, "relayout event wait failed");
            }
        }
        ++d->relayouts;
        d->bytes_sent += (int64_t)(16 * chunk) * ((1 << k) - 1);
        return QSV_OK;
    }
    if (int rc = sync_all(d)) return rc;
    for (int r = 0; r < d->P; ++r) {
        const int rs = s_value(r);
        for (int c = 0; c < (1 << k); ++c) {
            if (c == rs) continue;
            const int p = partner(r, c);
            if (p < r) continue;  // each unordered pair once
            qsv_state *A = d->shards[r], *B = d->shards[p];
            double2 *a = A->amps + (uint64_t)c * chunk, *b = B->amps + (uint64_t)rs * chunk;
            const size_t bytes = 16 * chunk;
            cudaSetDevice(A->device);
            char *stg = (char *)d->staging[r];
            for (size_t off = 0; off < bytes; off += d->piece_bytes) {
                const size_t w = std::min(d->piece_bytes, bytes - off);
                char *pa = (char *)a + off, *pb = (char *)b + off;
                if (cudaMemcpyAsync(stg, pa, w, cudaMemcpyDeviceToDevice, A->stream) != cudaSuccess ||
                    cudaMemcpyPeerAsync(pa, A->device, pb, B->device, w, A->stream) != cudaSuccess ||
                    cudaMemcpyPeerAsync(pb, B->device, stg, A->device, w, A->stream) != cudaSuccess)
                    return fail_code(QSV_ERR_CUDA, "relayout copy failed");
            }
        }
    }
    if (int rc = sync_all(d)) return rc;
    ++d->relayouts;
    d->bytes_sent += (int64_t)(16 * chunk) * ((1 << k) - 1);
    return QSV_OK;
}

int materialize(qsv_dist *d)
{
    if (!d->lazy) return QSV_OK;
    const uint64_t owner = d->basis >> d->n_local, local = d->basis & ((1ull << d->n_local) - 1);
    for (int r = 0; r < d->P; ++r) {
        qsv_state *s = d->shards[r];
        if ((uint64_t)r == owner) {
            if (int rc = qsv_set_basis(s, local)) return rc;
        } else {
            cudaSetDevice(s->device);
            if (cudaMemsetAsync(s->amps, 0, 16 * s->dim, s->stream) != cudaSuccess)
                return fail_code(QSV_ERR_CUDA, "shard zero fill failed");
        }
    }
    d->lazy = false;
    return QSV_OK;
}

int apply_segment_gates(qsv_dist *d, const Segment &seg, const int32_t *kinds, const double *values)
{
    const size_t L = seg.src.size();
    if (!L) return QSV_OK;
    std::vector<int32_t> sk(L);
    std::vector<double> sv(3 * L, 0.0);
    for (size_t j = 0; j < L; ++j) {
        const int64_t i = seg.src[j];
        if (i < 0) {
            sk[j] = kSwap;
        } else {
            sk[j] = kinds[i];
            for (int v = 0; v < 3; ++v) sv[3 * j + v] = values[3 * i + v];
        }
    }
    for (qsv_state *s : d->shards)
        if (int rc = qsv_apply_gates(s, (int64_t)L, sk.data(), seg.qubits.data(), sv.data(), nullptr)) return rc;
    return QSV_OK;
}

uint64_t phys_mask(const qsv_dist *d, uint64_t m)
{
    uint64_t out = 0;
    for (int q = 0; q < d->n; ++q)
        if ((m >> q) & 1ull) out |= 1ull << d->perm[q];
    return out;
}

}  // namespace
}  // namespace qsv

using namespace qsv;

extern "C" {

int qsv_dist_create(qsv_dist **out, int n_qubits, int n_ranks, const int *device_ids)
{
    std::lock_guard<std::recursive_mutex> lk(d_mu);
    if (!out) return fail_code(QSV_ERR_INVALID, "null output");
    *out = nullptr;
    if (n_ranks < 1 || (n_ranks & (n_ranks - 1))) return fail_code(QSV_ERR_INVALID, "rank count must be a power of two");
    int g = 0;
    while ((1 << g) < n_ranks) ++g;
    if (n_qubits - g < 2) return fail_code(QSV_ERR_INVALID, "too few local qubits per shard");
    if (n_qubits > kMaxQubits) return fail_code(QSV_ERR_RESOURCE, "qubit count out of range");
    qsv_dist *d = new qsv_dist;
    d->n = n_qubits;
    d->g = g;
    d->P = n_ranks;
    d->n_local = n_qubits - g;
    d->perm.resize(n_qubits);
    for (int q = 0; q < n_qubits; ++q) d->perm[q] = q;
    d->piece_bytes = std::min<size_t>(d->piece_bytes, (size_t)16 << (d->n_local > 1 ? d->n_local - 1 : 0));
    std::set<std::pair<int, int>> peer_done;
    for (int r = 0; r < n_ranks; ++r) {
        const int dev = device_ids ? device_ids[r] : 0;
        d->devices.push_back(dev);
        qsv_state *s = nullptr;
        if (int rc = qsv_create(&s, d->n_local, dev)) {
            qsv_dist_destroy(d);
            return rc;
        }
        d->shards.push_back(s);
        void *stg = nullptr;
        cudaSetDevice(dev);
        if (cudaMalloc(&stg, d->piece_bytes) != cudaSuccess) {
            cudaGetLastError();
            qsv_dist_destroy(d);
            return fail_code(QSV_ERR_NOMEM, "relayout staging allocation failed");
        }
        d->staging.push_back(stg);
        cudaEvent_t e1 = nullptr, e2 = nullptr;
        if (cudaEventCreateWithFlags(&e1, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&e2, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            qsv_dist_destroy(d);
            return fail_code(QSV_ERR_CUDA, "relayout event creation failed");
        }
        d->ev_ready.push_back(e1);
        d->ev_done.push_back(e2);
    }
    // peer access between distinct devices (NVLink / NVSwitch): the swap
    // kernels address the partner's shard directly; without it
    // cudaMemcpyPeerAsync still works, staged by the driver
    d->p2p = true;
    for (int a : d->devices)
        for (int b : d->devices)
            if (a != b && !peer_done.count({a, b})) {
                peer_done.insert({a, b});
                int can = 0;
                cudaDeviceCanAccessPeer(&can, a, b);
                if (can) {
                    cudaSetDevice(a);
                    const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
                    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) d->p2p = false;
                    cudaGetLastError();
                } else {
                    d->p2p = false;
                }
            }
    *out = d;
    return QSV_OK;
}

int qsv_dist_destroy(qsv_dist *d)
{
    std::lock_guard<std::recursive_mutex> lk(d_mu);
    if (!d) return QSV_OK;
    for (qsv_state *s : d->shards) qsv_destroy(s);
    for (size_t r = 0; r < d->staging.size(); ++r) {
        cudaSetDevice(d->devices[r]);
        cudaFree(d->staging[r]);
    }
    for (size_t r = 0; r < d->ev_ready.size(); ++r) {
        cudaSetDevice(d->devices[r]);
        cudaEventDestroy(d->ev_ready[r]);
        cudaEventDestroy(d->ev_done[r]);
    }
    delete d;
    return QSV_OK;
}

int qsv_dist_set_basis(qsv_dist *d, uint64_t index)
{
    std::lock_guard<std::recursive_mutex> lk(d_mu);
    if (!d) return fail_code(QSV_ERR_INVALID, "null handle");
    if (d->n < 64 && (index >> d->n)) return fail_code(QSV_ERR_INVALID, "basis index out of range");
    for (int q = 0; q < d->n; ++q) d->perm[q] = q;  // a fresh state: identity layout
    d->lazy = true;
    d->basis = index;
    return QSV_OK;
}

int qsv_dist_apply_gates(qsv_dist *d, int64_t n_gates, const int32_t *kinds, const int32_t *qubits,
                         const double *values)
{
    std::lock_guard<std::recursive_mutex> lk(d_mu);
    if (!d) return fail_code(QSV_ERR_INVALID, "null handle");
    if (n_gates < 0 || (n_gates > 0 && (!kinds || !qubits || !values)))
        return fail_code(QSV_ERR_INVALID, "bad gate arrays");
    for (int64_t i = 0; i < n_gates; ++i) {
        int gq[2];
        const int nq = gate_qubits(qubits, i, gq);
        for (int k = 0; k < nq; ++k)
            if (gq[k] < 0 || gq[k] >= d->n) return fail_code(QSV_ERR_INVALID, "gate qubit out of range");
        if (kinds[i] < 0 || kinds[i] >= K_COUNT) return fail_code(QSV_ERR_INVALID, "unknown gate kind");
    }
    if (int rc = materialize(d)) return rc;
    std::vector<Segment> segs;
    std::string err;
    std::vector<int> perm = d->perm;
    if (!plan_segments(n_gates, qubits, d->n, d->n_local, perm, segs, err))
        return fail_code(QSV_ERR_INVALID, err);
    for (const Segment &seg : segs) {
        if (int rc = apply_segment_gates(d, seg, kinds, values)) return rc;
        if (seg.has_relayout)
            if (int rc = relayout(d, seg.rl)) return rc;
    }
    d->perm = perm;
    return QSV_OK;
}

// distributed.py DistStateVector.expectation_terms: strings whose flip avoids
// the global bits run on every shard (a Z on a global bit is a per-rank
// sign); the others are localised by relayouts (the state is logically
// unchanged).  Partials are summed in ascending rank order (engine.py:199).
int qsv_dist_expectation(qsv_dist *d, int64_t S, const uint64_t *x, const uint64_t *y, const uint64_t *z,
                         const double *coef_re, const double *coef_im, double *out_re, double *out_im)
{
    std::lock_guard<std::recursive_mutex> lk(d_mu);
    if (!d || !out_re || !out_im) return fail_code(QSV_ERR_INVALID, "null argument");
    if (S < 0 || (S > 0 && (!x || !y || !z || !coef_re))) return fail_code(QSV_ERR_INVALID, "bad term arrays");
    const uint64_t allowed = d->n >= 64 ? ~0ull : ((1ull << d->n) - 1ull);
    for (int64_t t = 0; t < S; ++t) {
        if ((x[t] | y[t] | z[t]) & ~allowed) return fail_code(QSV_ERR_INVALID, "string index out of range");
        if (__builtin_popcountll(x[t] | y[t]) > d->n_local)
            return fail_code(QSV_ERR_INVALID, "Pauli string wider than the local qubits of a shard");
    }
    if (int rc = materialize(d)) return rc;
    const uint64_t lmask = (1ull << d->n_local) - 1ull;
    std::vector<double> pre(d->P, 0.0), pim(d->P, 0.0);
    std::vector<int64_t> remaining(S);
    for (int64_t t = 0; t < S; ++t) remaining[t] = t;
    while (!remaining.empty()) {
        std::vector<int64_t> loc, rest;
        for (int64_t t : remaining) {
            const uint64_t f = phys_mask(d, x[t] | y[t]);
            (f >> d->n_local ? rest : loc).push_back(t);
        }
        if (!loc.empty()) {
            const size_t L = loc.size();
            std::vector<uint64_t> lx(L), ly(L), lz(L), gz(L);
            std::vector<double> ones(L, 1.0), zeros(L, 0.0), per(L);
            for (size_t j = 0; j < L; ++j) {
                const int64_t t = loc[j];
                lx[j] = phys_mask(d, x[t]) & lmask;
                ly[j] = phys_mask(d, y[t]) & lmask;
                const uint64_t pz = phys_mask(d, z[t]);
                lz[j] = pz & lmask;
                gz[j] = pz >> d->n_local;
            }
            for (int r = 0; r < d->P; ++r) {
                double re = 0, im = 0;
                if (int rc = qsv_expectation(d->shards[r], (int64_t)L, lx.data(), ly.data(), lz.data(),
                                             ones.data(), zeros.data(), &re, &im, per.data(), nullptr))
                    return rc;
                for (size_t j = 0; j < L; ++j) {
                    const double v = (__builtin_popcountll(gz[j] & (uint64_t)r) & 1) ? -per[j] : per[j];
                    pre[r] += coef_re[loc[j]] * v;
                    pim[r] += (coef_im ? coef_im[loc[j]] : 0.0) * v;
                }
            }
        }
        remaining.swap(rest);
        if (remaining.empty()) break;
        // localise the first remaining flip (distributed.py plan_localize)
        std::vector<int> inv(d->n);
        for (int q = 0; q < d->n; ++q) inv[d->perm[q]] = q;
        const uint64_t f0 = x[remaining[0]] | y[remaining[0]];
        std::vector<int> bring;
        for (int q = 0; q < d->n; ++q)
            if (((f0 >> q) & 1ull) && d->perm[q] >= d->n_local) bring.push_back(q);
        std::vector<int> freq(d->n, 0);
        for (int64_t t : remaining)
            for (int q = 0; q < d->n; ++q) freq[q] += ((x[t] | y[t]) >> q) & 1ull;
        std::vector<int> cand;
        for (int p = 0; p < d->n_local; ++p)
            if (!((f0 >> inv[p]) & 1ull)) cand.push_back(inv[p]);
        std::sort(cand.begin(), cand.end(), [&](int a, int b) {
            if (freq[a] != freq[b]) return freq[a] < freq[b];
            return a < b;
        });
        if (cand.size() < bring.size()) return fail_code(QSV_ERR_INVALID, "cannot localise a Pauli string");
        std::vector<int> victims(cand.begin(), cand.begin() + bring.size());
        std::vector<std::pair<int, int>> swaps;
        move_victims(d->perm, inv, victims, d->n_local, swaps);
        if (!swaps.empty()) {
            Segment sw;
            for (auto &p : swaps) {
                sw.src.push_back(-1);
                sw.qubits.push_back(p.first);
                sw.qubits.push_back(p.second);
            }
            if (int rc = apply_segment_gates(d, sw, nullptr, nullptr)) return rc;
        }
        Relayout rl;
        for (int b : bring) rl.S.push_back(d->perm[b] - d->n_local);
        if (int rc = relayout(d, rl)) return rc;
        apply_relayout_to_map(d->perm, inv, bring, victims, d->n_local);
    }
    double re = 0.0, im = 0.0;
    for (int r = 0; r < d->P; ++r) {  // ascending rank order (engine.py:199)
        re += pre[r];
        im += pim[r];
    }
    *out_re = re;
    *out_im = im;
    return QSV_OK;
}

int qsv_dist_download(qsv_dist *d, double *host)
{
    std::lock_guard<std::recursive_mutex> lk(d_mu);
    if (!d || !host) return fail_code(QSV_ERR_INVALID, "null argument");
    if (int rc = materialize(d)) return rc;
    const uint64_t dim_local = 1ull << d->n_local, dim = 1ull << d->n;
    std::vector<double> phys(2 * dim);
    for (int r = 0; r < d->P; ++r)
        if (int rc = qsv_download(d->shards[r], phys.data() + 2 * (uint64_t)r * dim_local)) return rc;
    // logical index -> physical index through the qubit map
    for (uint64_t i = 0; i < dim; ++i) {
        uint64_t p = 0;
        for (int q = 0; q < d->n; ++q) p |= ((i >> q) & 1ull) << d->perm[q];
        host[2 * i] = phys[2 * p];
        host[2 * i + 1] = phys[2 * p + 1];
    }
    return QSV_OK;
}

int qsv_dist_p2p_info(const qsv_dist *d, int *p2p, int64_t *swap_launches)
{
    std::lock_guard<std::recursive_mutex> lk(d_mu);
    if (!d) return fail_code(QSV_ERR_INVALID, "null handle");
    if (p2p) *p2p = d->p2p ? 1 : 0;
    if (swap_launches) *swap_launches = d->swap_launches;
    return QSV_OK;
}

int qsv_dist_info(const qsv_dist *d, int *n_ranks, int *local_qubits, int64_t *relayouts,
                  int64_t *bytes_sent_per_rank, int32_t *perm)
{
    std::lock_guard<std::recursive_mutex> lk(d_mu);
    if (!d) return fail_code(QSV_ERR_INVALID, "null handle");
    if (n_ranks) *n_ranks = d->P;
    if (local_qubits) *local_qubits = d->n_local;
    if (relayouts) *relayouts = d->relayouts;
    if (bytes_sent_per_rank) *bytes_sent_per_rank = d->bytes_sent;
    if (perm)
        for (int q = 0; q < d->n; ++q) perm[q] = d->perm[q];
    return QSV_OK;
}

}  // extern "C"
