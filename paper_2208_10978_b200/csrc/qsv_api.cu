// qsv_api.cu -- the C ABI (include/qsv.h): handles, validation, program
// staging and launch sequencing.  Every compute entry point runs on the GPU;
// there is no CPU path.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>
#include <list>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/qsv.h"
#include "qsv_internal.h"
#include "qsv_planner.h"

namespace qsv {

namespace {

thread_local std::string g_err;
thread_local qsv_plan_stats g_last_stats{};
int64_t g_jit_launches = 0;  // specialised pass launches (debug / tests)

std::recursive_mutex g_mu;

struct DeviceCtx {
    bool init = false;
    cudaStream_t stream = nullptr;
    void *d_work = nullptr;
    size_t d_bytes = 0;
    void *h_stage = nullptr;
    size_t h_bytes = 0;
    cudaEvent_t stage_ev = nullptr;
    bool stage_pending = false;
    cudaStream_t copy_stream = nullptr;  // asynchronous downloads (lazily created)
};
DeviceCtx g_dev[64];

#define QSV_CUDA(call)                                                                   \
    do {                                                                                 \
        cudaError_t _e = (call);                                                         \
        if (_e != cudaSuccess)                                                           \
            return fail_code(QSV_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

int fail_code(int code, const std::string &msg)
{
    g_err = msg;
    return code;
}

int ctx_for(int device, DeviceCtx **out)
{
    if (device < 0 || device >= 64) return fail_code(QSV_ERR_INVALID, "device index out of range");
    DeviceCtx &c = g_dev[device];
    QSV_CUDA(cudaSetDevice(device));
    if (!c.init) {
        QSV_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
        QSV_CUDA(cudaEventCreateWithFlags(&c.stage_ev, cudaEventDisableTiming));
        c.init = true;
    }
    *out = &c;
    return QSV_OK;
}

constexpr size_t kBigWork = (size_t)1 << 30;

// Free a workspace that a large one-off request grew past 1 GiB, so a sample
// of a big state does not pin tens of GiB for the rest of the process.
int release_big_work(DeviceCtx &c, cudaStream_t st)
{
    if (c.d_bytes < kBigWork) return QSV_OK;
    QSV_CUDA(cudaStreamSynchronize(st));
    QSV_CUDA(cudaFree(c.d_work));
    c.d_work = nullptr;
    c.d_bytes = 0;
    return QSV_OK;
}

int ensure_work(DeviceCtx &c, cudaStream_t st, size_t bytes)
{
    if (c.d_bytes >= bytes) return QSV_OK;
    QSV_CUDA(cudaStreamSynchronize(st));
    if (c.d_work) QSV_CUDA(cudaFree(c.d_work));
    c.d_work = nullptr;
    // small requests grow with headroom; large ones (sampling a >= 27-qubit
    // state) are allocated exactly and released after use (release_big_work)
    size_t want = bytes >= kBigWork ? bytes : std::max<size_t>(bytes + bytes / 2, (size_t)1 << 20);
    if (cudaMalloc(&c.d_work, want) != cudaSuccess) {
        cudaGetLastError();
        c.d_bytes = 0;
        return fail_code(QSV_ERR_NOMEM, "device workspace allocation failed");
    }
    c.d_bytes = want;
    return QSV_OK;
}

int ensure_stage(DeviceCtx &c, size_t bytes)
{
    if (c.stage_pending) {
        QSV_CUDA(cudaEventSynchronize(c.stage_ev));
        c.stage_pending = false;
    }
    if (c.h_bytes >= bytes) return QSV_OK;
    if (c.h_stage) QSV_CUDA(cudaFreeHost(c.h_stage));
    c.h_stage = nullptr;
    size_t want = std::max<size_t>(bytes + bytes / 2, (size_t)1 << 20);
    if (cudaMallocHost(&c.h_stage, want) != cudaSuccess) {
        cudaGetLastError();
        c.h_bytes = 0;
        return fail_code(QSV_ERR_NOMEM, "pinned staging allocation failed");
    }
    c.h_bytes = want;
    return QSV_OK;
}

// Host blob assembled from several arrays; uploaded with one H2D copy.
struct Blob {
    std::vector<char> bytes;
    size_t add(const void *p, size_t n)
    {
        size_t off = (bytes.size() + 255) & ~(size_t)255;
        bytes.resize(off + n);
        if (n && p) std::memcpy(bytes.data() + off, p, n);
        return off;
    }
};

// Upload blob into the head of the device workspace; extra = trailing scratch.
int upload_blob(DeviceCtx &c, cudaStream_t st, const Blob &b, size_t extra, char **d_base,
                size_t *scratch_off)
{
    const size_t head = (b.bytes.size() + 255) & ~(size_t)255;
    int rc = ensure_work(c, st, head + extra + 256);
    if (rc) return rc;
    if (!b.bytes.empty()) {
        rc = ensure_stage(c, b.bytes.size());
        if (rc) return rc;
        std::memcpy(c.h_stage, b.bytes.data(), b.bytes.size());
        QSV_CUDA(cudaMemcpyAsync(c.d_work, c.h_stage, b.bytes.size(), cudaMemcpyHostToDevice, st));
        QSV_CUDA(cudaEventRecord(c.stage_ev, st));
        c.stage_pending = true;
    }
    *d_base = (char *)c.d_work;
    *scratch_off = head;
    return QSV_OK;
}

int check_state(const qsv_state *s)
{
    if (!s || !s->amps) return fail_code(QSV_ERR_INVALID, "null or destroyed state handle");
    return QSV_OK;
}

// Order work that modifies (or frees) s after its in-flight asynchronous
// download: a device-side wait on the state's stream, or (host) a blocking
// wait for the copy itself.
int settle(qsv_state *s, bool host = false)
{
    if (!s || !s->dl_pending) return QSV_OK;
    if (host) {
        QSV_CUDA(cudaEventSynchronize(s->dl_done));
    } else {
        QSV_CUDA(cudaStreamWaitEvent(s->stream, s->dl_done, 0));
    }
    s->dl_pending = false;
    return QSV_OK;
}

// QSV_HOST_PROFILE=1: per-phase host time of an API call on stderr.
struct HostProfile {
    const char *what;
    bool on;
    std::chrono::steady_clock::time_point t0, t;
    std::string line;
    explicit HostProfile(const char *w) : what(w)
    {
        const char *e = getenv("QSV_HOST_PROFILE");
        on = e && e[0] == '1';
        if (on) t0 = t = std::chrono::steady_clock::now();
    }
    void mark(const char *phase)
    {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        char buf[96];
        snprintf(buf, sizeof(buf), " %s %.1f us", phase,
                 std::chrono::duration<double, std::micro>(now - t).count());
        line += buf;
        t = now;
    }
    ~HostProfile()
    {
        if (on)
            fprintf(stderr, "qsv host %s:%s (total %.1f us)\n", what, line.c_str(),
                    std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0)
                        .count());
    }
};

// Specialised sources of a cached program and their loaded modules (built on
// the first specialised run, reused by every later one).
struct JitCache {
    int device = -1;
    std::vector<std::string> src;
    std::vector<const void *> mod;
    // fast path once every pass has a module: per-pass geometry tables and
    // parameter window, so a run uploads only tables + parameters
    bool all_jit = false;
    std::vector<std::vector<uint64_t>> offhi;
    std::vector<std::vector<int32_t>> comp;
    std::vector<int> p_lo, npar;
    // OP_GMAT tables filled on the device in the fast path: per table its
    // pass and offset inside that pass's parameter window, and the groups'
    // concatenated yF bytes
    std::vector<int> gmat_pass, gmat_rel, gmat_yf;
    std::vector<uint8_t> yF;
    // per pass: window ranges [a, b) (doubles) NOT covered by GMAT tables --
    // the only parameters the host must upload when the tables are filled
    // on the device (an all-GMAT window lives in device scratch only)
    std::vector<std::vector<std::pair<int, int>>> host_ranges;
};

bool fast_path(const qsv_state *s, const ProgramTemplate &t, const JitCache *jc, int uses)
{
    return jc && jc->all_jit && jc->device == s->device && jc->src.size() == t.passes.size() &&
           jit_enabled(s->n, uses);
}

// Planner / sweep knobs that change a plan: part of every cache key, so a
// process that changes one (tests pin tile geometries this way) never reuses a
// plan made under another setting.
std::string planner_knobs()
{
    static const char *names[] = {"QSV_MIN_CONTIG", "QSV_FUSE_QUBITS", "QSV_PASS_PARAM_CAP",
                                  "QSV_PASS_COST_CAP", "QSV_SCHED_SEEDS", "QSV_SCHED",
                                  "QSV_SCHED_WINDOW", "QSV_PHASE_DEFER", "QSV_WARP_LOCAL",
                                  "QSV_BLOCK_PARTITION", "QSV_INREG_PERMS", "QSV_SWEEP_TERMS",
                                  "QSV_SWEEP_SHARE", "QSV_JIT", "QSV_JIT_MIN_QUBITS", "QSV_TILE_BITS",
                                  "QSV_U3_NORM", "QSV_SWEEP_FUSE1", "QSV_SWEEP_COSET",
                                  "QSV_SWEEP_WARPS", "QSV_COMPACT_GMAT", "QSV_PASS_TMA",
                                  "QSV_CZ_DEFER", "QSV_SWEEP_ONETILE"};
    std::string k;
    for (const char *nm : names) {
        const char *v = getenv(nm);
        k += v ? v : "-";
        k += '|';
    }
    if (plain_u3()) k += "plain";
    return k;
}

struct PlainU3Scope {
    PlainU3Scope() { set_plain_u3(true); }
    ~PlainU3Scope() { set_plain_u3(false); }
};

// Cache of structural gate plans.
struct CacheEntry {
    uint64_t hash;
    int n;
    std::string knobs;
    std::vector<int32_t> kinds, qubits;
    ProgramTemplate tpl;
    int uses = 0;  // runs of this structure (hot programs get specialised passes)
    JitCache jc;
};
std::list<CacheEntry> g_cache;
constexpr size_t kCacheMax = 8;

struct ExpCacheEntry {
    uint64_t hash;
    int n;
    std::string knobs;
    bool jit = false;
    std::vector<std::string> jit_src;  // per sweep ("" = interpreted)
    std::vector<uint64_t> x, y, z;
    std::vector<SweepPlan> plan;
};
std::list<ExpCacheEntry> g_exp_cache;

uint64_t hash_masks(int n, int64_t S, const uint64_t *x, const uint64_t *y, const uint64_t *z)
{
    uint64_t h = 0xcbf29ce484222325ull ^ (uint64_t)n;
    for (int64_t t = 0; t < S; ++t) {
        uint64_t v[3] = {x[t], y[t], z[t]};
        for (uint64_t w : v) {
            h ^= w + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
            h *= 1099511628211ull;
        }
    }
    return h;
}

// Parameter doubles an op reads (for pass-local rebasing).
int op_param_count(const OpRec &op)
{
    switch (op.type) {
        case OP_U1: return 8;
        case OP_U1C: return 16;
        case OP_U2: return 32;
        case OP_DIAG1: return 4;
        case OP_GMAT: return 16 << (__builtin_popcount(op.f) - 1);
        default: return 0;
    }
}

// Pass-local program of pass k (op / rot / param indices rebased to the
// pass) and its specialised source; shared by run_template and the debug
// export.  Returns false for global / tiny passes.
static bool pass_local(const ProgramTemplate &t, size_t k, std::vector<OpRec> &lops,
                       std::vector<BlockRec> &lblk, int &r_lo, int &r_hi, int &p_lo, int &p_hi)
{
    const PassPlan &p = t.passes[k];
    if (p.global || p.geom.m < kBlockBits + 1) return false;
    r_lo = INT32_MAX, r_hi = 0, p_lo = INT32_MAX, p_hi = 0;
    for (int i = p.op_begin; i < p.op_end; ++i) {
        const OpRec &op = t.ops[i];
        if (op.r1 > op.r0) {
            r_lo = std::min(r_lo, op.r0);
            r_hi = std::max(r_hi, op.r1);
        }
        const int np = op_param_count(op);
        if (np) {
            p_lo = std::min(p_lo, op.p);
            p_hi = std::max(p_hi, op.p + np);
        }
    }
    if (r_lo == INT32_MAX) r_lo = r_hi = 0;
    if (p_lo == INT32_MAX) p_lo = p_hi = 0;
    p_lo &= ~3;  // keep 32 B alignment of matrices
    lops.assign(t.ops.begin() + p.op_begin, t.ops.begin() + p.op_end);
    for (OpRec &op : lops) {
        if (op.r1 > op.r0) {
            op.r0 -= r_lo;
            op.r1 -= r_lo;
        }
        if (op_param_count(op)) op.p -= p_lo;
    }
    lblk.assign(t.blocks.begin() + p.block_begin, t.blocks.begin() + p.block_end);
    for (BlockRec &bl : lblk) {
        bl.op0 -= p.op_begin;
        bl.op1 -= p.op_begin;
    }
    return true;
}

// A cached program whose every pass is specialised: upload each pass's
// geometry tables and parameter window, copy-and-launch.
int run_template_jit(qsv_state *s, ProgramTemplate &t, const std::vector<double> &params,
                     JitCache &jc, DeviceCtx &c, bool gmats_on_device, uint64_t basis)
{
    HostProfile prof("run_template_jit");
    Blob b;
    const size_t np = t.passes.size();
    std::vector<size_t> o_off(np), o_comp(np), o_par(np);
    std::vector<char> in_scratch(np, 0);
    size_t scratch_bytes = 0;
    for (size_t k = 0; k < np; ++k) {
        if (!jc.mod[k]) continue;
        o_off[k] = b.add(jc.offhi[k].data(), jc.offhi[k].size() * sizeof(uint64_t));
        o_comp[k] = b.add(jc.comp[k].data(), jc.comp[k].size() * sizeof(int32_t));
        if (gmats_on_device && jc.host_ranges[k].empty()) {  // tables only: device scratch
            in_scratch[k] = 1;
            o_par[k] = scratch_bytes;  // relative to the scratch base, fixed below
            scratch_bytes += ((size_t)jc.npar[k] * 8 + 255) & ~(size_t)255;
        } else if (gmats_on_device) {  // upload only the non-table parameters
            o_par[k] = b.add(nullptr, (size_t)jc.npar[k] * sizeof(double));
            for (const auto &rg : jc.host_ranges[k])
                std::memcpy(b.bytes.data() + o_par[k] + (size_t)rg.first * 8,
                            params.data() + jc.p_lo[k] + rg.first, (size_t)(rg.second - rg.first) * 8);
        } else {
            o_par[k] = b.add(params.data() + jc.p_lo[k], (size_t)jc.npar[k] * sizeof(double));
        }
    }
    const int ng = gmats_on_device ? (int)t.gfills.size() : 0;
    size_t o_jobs = 0, o_cs = 0, o_q = 0, o_yf = 0;
    if (ng) {
        std::vector<double> cs(2 * t.rots.size());
        std::vector<int32_t> q(t.rots.size());
        for (size_t r = 0; r < t.rots.size(); ++r) {
            cs[2 * r] = t.rots[r].c;
            cs[2 * r + 1] = t.rots[r].s;
            q[r] = t.rots[r].q;
        }
        o_cs = b.add(cs.data(), cs.size() * sizeof(double));
        o_q = b.add(q.data(), q.size() * sizeof(int32_t));
        o_yf = b.add(jc.yF.data(), jc.yF.size());
        o_jobs = b.add(nullptr, (size_t)ng * sizeof(GmatJob));  // filled once offsets are final
    }
    // upload_blob puts the scratch right after the blob (256-B aligned)
    const size_t scratch_base = (b.bytes.size() + 255) & ~(size_t)255;
    for (size_t k = 0; k < np; ++k)
        if (in_scratch[k]) o_par[k] += scratch_base;
    for (int i = 0; i < ng; ++i) {
        const GmatFill &g = t.gfills[i];
        const GmatJob job{(uint64_t)(o_par[jc.gmat_pass[i]] + (size_t)jc.gmat_rel[i] * 8), g.r0, g.r1,
                          g.F, g.H, g.w, jc.gmat_yf[i]};
        std::memcpy(b.bytes.data() + o_jobs + (size_t)i * sizeof(GmatJob), &job, sizeof(GmatJob));
    }
    prof.mark("blob");
    char *d = nullptr;
    size_t scratch = 0;
    if (int rc = upload_blob(c, s->stream, b, scratch_bytes, &d, &scratch)) return rc;
    if (scratch != scratch_base) return fail_code(QSV_ERR_CUDA, "unexpected workspace layout");
    if (ng)
        QSV_CUDA(launch_gmat_fill(d, (const GmatJob *)(d + o_jobs), ng, (const double2 *)(d + o_cs),
                                  (const int32_t *)(d + o_q), (const uint8_t *)(d + o_yf), s->stream));
    prof.mark("upload");
    bool first = true;
    for (size_t k = 0; k < np; ++k) {
        const PassPlan &p = t.passes[k];
        if (!jc.mod[k]) continue;
        if (!jit_launch_module(jc.mod[k], s->amps, dims_of(p.geom), (const uint64_t *)(d + o_off[k]),
                               (const int32_t *)(d + o_comp[k]), (const double *)(d + o_par[k]),
                               jc.npar[k],
                               (int)std::min<uint64_t>(1ull << p.geom.ncomp, (uint64_t)num_sms(s->device)),
                               s->stream, first ? basis : ~0ull))
            return fail_code(QSV_ERR_CUDA, "specialised pass launch failed");
        first = false;
        ++g_jit_launches;
    }
    if (first && basis != ~0ull) QSV_CUDA(launch_set_basis(s->amps, s->dim, basis, s->stream));
    prof.mark("launch");
    return QSV_OK;
}

// gmats_on_device: params lack the OP_GMAT tables (materialize_params with
// with_gmats = false); only valid when fast_path() holds.
// basis != ~0: the state is first set to |basis> -- fused into the first
// pass when that pass is specialised, else a set_basis launch.
int run_template(qsv_state *s, ProgramTemplate &t, const std::vector<double> &params, int uses = 0,
                 JitCache *jc = nullptr, bool gmats_on_device = false, uint64_t basis = ~0ull)
{
    DeviceCtx *c = nullptr;
    int rc = ctx_for(s->device, &c);
    if (rc) return rc;
    if (fast_path(s, t, jc, uses))
        return run_template_jit(s, t, params, *jc, *c, gmats_on_device, basis);
    HostProfile prof("run_template");
    Blob b;
    // global (shared) arrays for the legacy / fallback kernels
    const size_t o_ops = b.add(t.ops.data(), t.ops.size() * sizeof(OpRec));
    const size_t o_rots = b.add(t.rots.data(), t.rots.size() * sizeof(RotRec));
    const size_t o_par = b.add(params.data(), params.size() * sizeof(double));
    struct PassOff { size_t off, comp, blk, ops, rots, par; int nblk, nops, nrots, npar, par_lo; bool lite; };
    std::vector<PassOff> po(t.passes.size());
    const bool jit = jit_enabled(s->n, uses);
    JitCache local;
    if (!jc) jc = &local;
    const bool jit_cached = jit && jc->device == s->device && jc->src.size() == t.passes.size();
    if (jit && !jit_cached) {
        jc->device = -1;
        jc->src.assign(t.passes.size(), std::string());
        jc->mod.assign(t.passes.size(), nullptr);
    }
    std::vector<std::string> &jit_src = jc->src;
    {
        std::vector<uint64_t> offhi;
        std::vector<int32_t> comp;
        std::vector<OpRec> lops;
        std::vector<BlockRec> lblk;
        for (size_t k = 0; k < t.passes.size(); ++k) {
            const PassPlan &p = t.passes[k];
            PassOff &o = po[k];
            o = PassOff{};
            if (p.global) continue;
            geom_tables(p.geom, offhi, comp, &t.passes[k]);
            o.off = b.add(offhi.data(), offhi.size() * sizeof(uint64_t));
            o.comp = b.add(comp.data(), comp.size() * sizeof(int32_t));
            int r_lo, r_hi, p_lo, p_hi;
            if (!pass_local(t, k, lops, lblk, r_lo, r_hi, p_lo, p_hi)) continue;
            o.lite = true;
            for (const OpRec &op : lops)
                if (op.type == OP_U2) o.lite = false;
            for (const BlockRec &bl : lblk)
                if (bl.kind != 0) o.lite = false;
            o.nblk = (int)lblk.size();
            o.nops = (int)lops.size();
            o.nrots = r_hi - r_lo;
            o.npar = p_hi - p_lo;
            o.par_lo = p_lo;
            if (jit && !jit_cached)
                jit_source(p.geom, lblk.data(), o.nblk, lops.data(), t.rots.data() + r_lo, o.npar,
                           jit_src[k]);
            o.blk = b.add(lblk.data(), lblk.size() * sizeof(BlockRec));
            o.ops = b.add(lops.data(), lops.size() * sizeof(OpRec));
            o.rots = b.add(t.rots.data() + r_lo, (size_t)o.nrots * sizeof(RotRec));
            o.par = b.add(params.data() + p_lo, (size_t)o.npar * sizeof(double));
        }
    }
    prof.mark("blob");
    char *d = nullptr;
    size_t scratch = 0;
    rc = upload_blob(*c, s->stream, b, 0, &d, &scratch);
    if (rc) return rc;
    prof.mark("upload");
    if (jit && !jit_cached) {
        std::vector<const std::string *> srcs;
        for (const std::string &src : jit_src)
            if (!src.empty()) srcs.push_back(&src);
        std::string err;
        if (!srcs.empty() && jit_prepare(s->device, srcs, err) && getenv("QSV_JIT_VERBOSE"))
            fprintf(stderr, "qsv jit: %s\n", err.c_str());
        for (size_t k = 0; k < jit_src.size(); ++k)
            jc->mod[k] = jit_src[k].empty() ? nullptr : jit_module(s->device, jit_src[k]);
        jc->device = s->device;
        // every pass that does work specialised (no global / small-tile /
        // fallback passes): later runs take run_template_jit
        bool all = true;
        for (size_t k = 0; k < t.passes.size(); ++k) {
            const PassPlan &p = t.passes[k];
            const bool idle = p.op_end <= p.op_begin && !p.map_permuted;
            if (!idle && (p.global || !jc->mod[k])) all = false;
            if (idle && jc->mod[k]) all = false;  // keep the general path's semantics
        }
        if (all) {
            jc->offhi.assign(t.passes.size(), {});
            jc->comp.assign(t.passes.size(), {});
            jc->p_lo.assign(t.passes.size(), 0);
            jc->npar.assign(t.passes.size(), 0);
            for (size_t k = 0; k < t.passes.size(); ++k) {
                if (!jc->mod[k]) continue;
                geom_tables(t.passes[k].geom, jc->offhi[k], jc->comp[k], &t.passes[k]);
                jc->p_lo[k] = (int)(po[k].par_lo);
                jc->npar[k] = po[k].npar;
            }
            // the pass window holding each OP_GMAT table
            jc->gmat_pass.assign(t.gfills.size(), -1);
            jc->gmat_rel.assign(t.gfills.size(), 0);
            jc->gmat_yf.assign(t.gfills.size(), 0);
            jc->yF.clear();
            for (size_t i = 0; i < t.gfills.size(); ++i) {
                const GmatFill &g = t.gfills[i];
                const int len = 16 << (g.w - 1);
                for (size_t k = 0; k < t.passes.size(); ++k)
                    if (jc->mod[k] && g.offset >= jc->p_lo[k] &&
                        g.offset + len <= jc->p_lo[k] + jc->npar[k]) {
                        jc->gmat_pass[i] = (int)k;
                        jc->gmat_rel[i] = g.offset - jc->p_lo[k];
                        break;
                    }
                if (jc->gmat_pass[i] < 0) all = false;
                jc->gmat_yf[i] = (int)jc->yF.size();
                jc->yF.insert(jc->yF.end(), g.yF.begin(), g.yF.end());
            }
            // window ranges not covered by tables
            jc->host_ranges.assign(t.passes.size(), {});
            for (size_t k = 0; k < t.passes.size() && all; ++k) {
                if (!jc->mod[k]) continue;
                std::vector<char> cov(jc->npar[k], 0);
                for (size_t i = 0; i < t.gfills.size(); ++i)
                    if (jc->gmat_pass[i] == (int)k)
                        std::fill(cov.begin() + jc->gmat_rel[i],
                                  cov.begin() + jc->gmat_rel[i] + (16 << (t.gfills[i].w - 1)), 1);
                for (int a = 0; a < jc->npar[k];) {
                    if (cov[a]) { ++a; continue; }
                    int e = a;
                    while (e < jc->npar[k] && !cov[e]) ++e;
                    jc->host_ranges[k].push_back({a, e});
                    a = e;
                }
            }
        }
        jc->all_jit = all;
    }
    const OpRec *d_ops = (const OpRec *)(d + o_ops);
    const RotRec *d_rots = (const RotRec *)(d + o_rots);
    const double *d_par = (const double *)(d + o_par);
    // the basis state can be synthesised by the first pass that runs only if
    // that pass is specialised
    size_t k_first = t.passes.size();
    for (size_t k = 0; k < t.passes.size(); ++k) {
        const PassPlan &p = t.passes[k];
        if (p.op_end > p.op_begin || p.map_permuted) {
            k_first = k;
            break;
        }
    }
    if (basis != ~0ull &&
        !(k_first < t.passes.size() && jit && jc->mod[k_first] && !t.passes[k_first].global)) {
        QSV_CUDA(launch_set_basis(s->amps, s->dim, basis, s->stream));
        basis = ~0ull;
    }
    for (size_t k = 0; k < t.passes.size(); ++k) {
        const PassPlan &p = t.passes[k];
        const PassOff &o = po[k];
        // a pass made only of permutation gates has no blocks but a permuted
        // store map: it still has to run (load -> store through the map)
        if (p.op_end <= p.op_begin && !p.map_permuted) continue;
        if (p.global) {
            for (int i = p.op_begin; i < p.op_end; ++i) {
                const OpRec &op = t.ops[i];
                QSV_CUDA(launch_rot_global(s->amps, s->n, p.flip, d_rots + op.r0, op.r1 - op.r0,
                                           s->stream));
            }
        } else {
            bool done = false;
            if (jit && jc->mod[k]) {
                done = jit_launch_module(jc->mod[k], s->amps, dims_of(p.geom),
                                         (const uint64_t *)(d + o.off), (const int32_t *)(d + o.comp),
                                         (const double *)(d + o.par), o.npar,
                                         (int)std::min<uint64_t>(1ull << p.geom.ncomp,
                                                                 (uint64_t)num_sms(s->device)),
                                         s->stream, k == k_first ? basis : ~0ull);
                if (done) ++g_jit_launches;
            }
            if (k == k_first && basis != ~0ull) {  // not synthesised by a specialised pass
                if (!done) QSV_CUDA(launch_set_basis(s->amps, s->dim, basis, s->stream));
                basis = ~0ull;
            }
            if (done) {
            } else if (p.geom.m >= kBlockBits + 1) {
                QSV_CUDA(launch_tile_blocks(s->amps, dims_of(p.geom), (const uint64_t *)(d + o.off),
                                            (const int32_t *)(d + o.comp), (const BlockRec *)(d + o.blk),
                                            o.nblk, (const OpRec *)(d + o.ops), o.nops,
                                            (const RotRec *)(d + o.rots), o.nrots,
                                            (const double *)(d + o.par), o.npar, o.lite, s->stream));
            } else {
                QSV_CUDA(launch_tile_pass(s->amps, dims_of(p.geom), (const uint64_t *)(d + o.off),
                                          (const int32_t *)(d + o.comp), d_ops + p.op_begin,
                                          p.op_end - p.op_begin, d_rots, d_par, s->stream));
            }
        }
    }
    prof.mark("launch");
    return QSV_OK;
}

void fill_stats(const ProgramTemplate &t, bool hit, qsv_plan_stats *out)
{
    qsv_plan_stats st{};
    st.n_input_ops = t.n_input;
    st.n_rotations = t.n_rotations;
    st.n_items = t.n_items;
    st.n_passes = (int64_t)t.passes.size();
    st.n_fallback = t.n_fallback;
    st.tile_bits = t.m;
    st.cache_hit = hit ? 1 : 0;
    g_last_stats = st;
    if (out) *out = st;
}

}  // namespace

void set_error(const std::string &msg) { g_err = msg; }
int fail(const std::string &msg) { return fail_code(QSV_ERR_INVALID, msg); }

}  // namespace qsv

using namespace qsv;

extern "C" {

int qsv_abi_version(void) { return QSV_ABI_VERSION; }

const char *qsv_last_error(void) { return g_err.c_str(); }

int qsv_device_count(int *out)
{
    if (!out) return fail_code(QSV_ERR_INVALID, "null output");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        *out = 0;
        return fail_code(QSV_ERR_CUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    }
    *out = n;
    return QSV_OK;
}

int qsv_mem_info(int device, uint64_t *free_bytes, uint64_t *total_bytes)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!free_bytes || !total_bytes) return fail_code(QSV_ERR_INVALID, "null output");
    if (device < 0 || device >= 64) return fail_code(QSV_ERR_INVALID, "device index out of range");
    QSV_CUDA(cudaSetDevice(device));
    size_t f = 0, t = 0;
    QSV_CUDA(cudaMemGetInfo(&f, &t));
    *free_bytes = f;
    *total_bytes = t;
    return QSV_OK;
}

int qsv_create(qsv_state **out, int n_qubits, int device)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!out) return fail_code(QSV_ERR_INVALID, "null output");
    *out = nullptr;
    if (n_qubits < 1 || n_qubits > kMaxQubits)
        return fail_code(QSV_ERR_RESOURCE, "qubit count out of range 1.." + std::to_string(kMaxQubits));
    DeviceCtx *c = nullptr;
    int rc = ctx_for(device, &c);
    if (rc) return rc;
    qsv_state *s = new qsv_state();
    s->n = n_qubits;
    s->device = device;
    s->dim = 1ull << n_qubits;
    s->stream = c->stream;
    const size_t bytes = (size_t)16 * s->dim;
    if (cudaMalloc((void **)&s->amps, bytes) != cudaSuccess) {
        cudaGetLastError();
        delete s;
        return fail_code(QSV_ERR_NOMEM, "cannot allocate " + std::to_string(bytes) +
                                            " bytes of device memory for the state");
    }
    *out = s;
    return QSV_OK;
}

int qsv_destroy(qsv_state *s)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!s) return QSV_OK;
    if (s->amps) {
        cudaSetDevice(s->device);
        settle(s, true);
        cudaStreamSynchronize(s->stream);
        cudaFree(s->amps);
        s->amps = nullptr;
    }
    if (s->dl_done) cudaEventDestroy(s->dl_done);
    delete s;
    return QSV_OK;
}

int qsv_n_qubits(const qsv_state *s, int *out)
{
    if (int rc = check_state(s)) return rc;
    *out = s->n;
    return QSV_OK;
}

// Every state keeps the device's library stream (shared scratch, pinned
// staging and __constant__ banks are ordered by it); a caller's stream is
// joined by an event fence instead of replacing it.
static int64_t g_swap_launches = 0;  // qsv_swap_peer kernels

// ---- cross-process relayouts (distributed.py over torch.distributed) --------
// A rank exports its shard with a CUDA IPC handle; its partners map it and
// swap chunks with it in place through the same swap kernel as qsv_dist
// (NVLink / NVSwitch P2P between GPUs of one node; plain device memory when
// two processes share a GPU).  The caller orders the swap against the
// partner's work (distributed.py: stream sync + barrier on both sides).

int qsv_ipc_get_handle(const qsv_state *s, void *handle)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(s)) return rc;
    if (!handle) return fail_code(QSV_ERR_INVALID, "null handle buffer");
    QSV_CUDA(cudaSetDevice(s->device));
    cudaIpcMemHandle_t h;
    QSV_CUDA(cudaIpcGetMemHandle(&h, s->amps));
    static_assert(sizeof(h) == QSV_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle, &h, sizeof(h));
    return QSV_OK;
}

int qsv_ipc_open(int device, const void *handle, void **peer_base)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!handle || !peer_base) return fail_code(QSV_ERR_INVALID, "null argument");
    *peer_base = nullptr;
    QSV_CUDA(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    QSV_CUDA(cudaIpcOpenMemHandle(peer_base, h, cudaIpcMemLazyEnablePeerAccess));
    return QSV_OK;
}

int qsv_ipc_close(int device, void *peer_base)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!peer_base) return QSV_OK;
    QSV_CUDA(cudaSetDevice(device));
    QSV_CUDA(cudaIpcCloseMemHandle(peer_base));
    return QSV_OK;
}

int qsv_swap_peer(qsv_state *s, uint64_t local_offset, void *peer_base, uint64_t peer_offset, uint64_t n)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(s)) return rc;
    if (!peer_base) return fail_code(QSV_ERR_INVALID, "null peer pointer");
    if (local_offset > s->dim || n > s->dim - local_offset)
        return fail_code(QSV_ERR_INVALID, "swap range outside the state");
    QSV_CUDA(cudaSetDevice(s->device));
    if (int rc = settle(s)) return rc;
    QSV_CUDA(launch_swap_chunks(s->amps + local_offset, (double2 *)peer_base + peer_offset, n,
                                num_sms(s->device), s->stream));
    ++g_swap_launches;
    return QSV_OK;
}

int qsv_swap_info(int64_t *launches)
{
    if (!launches) return fail_code(QSV_ERR_INVALID, "null output");
    *launches = g_swap_launches;
    return QSV_OK;
}

int qsv_set_stream(qsv_state *s, void *stream)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(s)) return rc;
    DeviceCtx *c = nullptr;
    if (int rc = ctx_for(s->device, &c)) return rc;
    if (!stream || (cudaStream_t)stream == c->stream) return QSV_OK;
    cudaEvent_t ev;
    QSV_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    QSV_CUDA(cudaEventRecord(ev, (cudaStream_t)stream));
    QSV_CUDA(cudaStreamWaitEvent(c->stream, ev, 0));
    QSV_CUDA(cudaEventDestroy(ev));  // released once the wait has been satisfied
    return QSV_OK;
}

int qsv_get_stream(const qsv_state *s, void **stream)
{
    if (int rc = check_state(s)) return rc;
    *stream = (void *)s->stream;
    return QSV_OK;
}

int qsv_device_ptr(const qsv_state *s, void **ptr)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(s)) return rc;
    // the caller may write through the pointer: no copy may still be reading
    if (int rc = settle(const_cast<qsv_state *>(s), true)) return rc;
    *ptr = (void *)s->amps;
    return QSV_OK;
}

int qsv_synchronize(qsv_state *s)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(s)) return rc;
    QSV_CUDA(cudaSetDevice(s->device));
    QSV_CUDA(cudaStreamSynchronize(s->stream));
    if (int rc = settle(s, true)) return rc;
    return QSV_OK;
}

int qsv_copy(qsv_state *dst, const qsv_state *src)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(dst)) return rc;
    if (int rc = check_state(src)) return rc;
    if (dst->n != src->n) return fail_code(QSV_ERR_INVALID, "state qubit counts differ");
    QSV_CUDA(cudaSetDevice(dst->device));
    if (dst == src) return QSV_OK;
    if (int rc = settle(dst)) return rc;
    QSV_CUDA(cudaMemcpyAsync(dst->amps, src->amps, 16 * dst->dim, cudaMemcpyDeviceToDevice,
                             dst->stream));
    return QSV_OK;
}

int qsv_embed_parity(qsv_state *dst, const qsv_state *half, uint64_t wlow, int cls)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(dst)) return rc;
    if (int rc = check_state(half)) return rc;
    if (dst->n != half->n + 1) return fail_code(QSV_ERR_INVALID, "half state must have one qubit less");
    if (wlow >> half->n) return fail_code(QSV_ERR_INVALID, "functional has bits beyond the half state");
    if (cls != 0 && cls != 1) return fail_code(QSV_ERR_INVALID, "class must be 0 or 1");
    if (dst == half) return fail_code(QSV_ERR_INVALID, "in-place embedding");
    QSV_CUDA(cudaSetDevice(dst->device));
    if (int rc = settle(dst)) return rc;
    QSV_CUDA(launch_embed_parity(dst->amps, half->amps, dst->n, wlow, (uint32_t)cls, num_sms(dst->device),
                                 dst->stream));
    return QSV_OK;
}

int qsv_set_basis(qsv_state *s, uint64_t index)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(s)) return rc;
    if (index >= s->dim) return fail_code(QSV_ERR_INVALID, "basis index out of range");
    QSV_CUDA(cudaSetDevice(s->device));
    if (int rc = settle(s)) return rc;
    QSV_CUDA(launch_set_basis(s->amps, s->dim, index, s->stream));
    return QSV_OK;
}

int qsv_upload(qsv_state *s, const double *host)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(s)) return rc;
    if (!host) return fail_code(QSV_ERR_INVALID, "null host buffer");
    QSV_CUDA(cudaSetDevice(s->device));
    if (int rc = settle(s)) return rc;
    QSV_CUDA(cudaMemcpyAsync(s->amps, host, 16 * s->dim, cudaMemcpyHostToDevice, s->stream));
    QSV_CUDA(cudaStreamSynchronize(s->stream));
    return QSV_OK;
}

int qsv_download(const qsv_state *s, double *host)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(s)) return rc;
    if (!host) return fail_code(QSV_ERR_INVALID, "null host buffer");
    QSV_CUDA(cudaSetDevice(s->device));
    QSV_CUDA(cudaMemcpyAsync(host, s->amps, 16 * s->dim, cudaMemcpyDeviceToHost, s->stream));
    QSV_CUDA(cudaStreamSynchronize(s->stream));
    return QSV_OK;
}

int qsv_download_async(qsv_state *s, double *host)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(s)) return rc;
    if (!host) return fail_code(QSV_ERR_INVALID, "null host buffer");
    DeviceCtx *c = nullptr;
    if (int rc = ctx_for(s->device, &c)) return rc;
    if (!c->copy_stream) QSV_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    if (!s->dl_done) QSV_CUDA(cudaEventCreateWithFlags(&s->dl_done, cudaEventDisableTiming));
    // copy stream: after the state's queued work, then the copy, then dl_done
    QSV_CUDA(cudaEventRecord(s->dl_done, s->stream));
    QSV_CUDA(cudaStreamWaitEvent(c->copy_stream, s->dl_done, 0));
    QSV_CUDA(cudaMemcpyAsync(host, s->amps, 16 * s->dim, cudaMemcpyDeviceToHost, c->copy_stream));
    QSV_CUDA(cudaEventRecord(s->dl_done, c->copy_stream));
    s->dl_pending = true;
    return QSV_OK;
}

int qsv_download_wait(qsv_state *s)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(s)) return rc;
    QSV_CUDA(cudaSetDevice(s->device));
    return settle(s, true);
}

static int validate_gates(const qsv_state *s, int64_t n, const int32_t *kinds,
                          const int32_t *qubits)
{
    for (int64_t i = 0; i < n; ++i) {
        const int k = kinds[i];
        if (k < 0 || k >= K_COUNT)
            return fail_code(QSV_ERR_INVALID, "unknown gate kind code " + std::to_string(k));
        const bool two = (k == K_CNOT || k == K_SWAP || k == K_CU3);
        const int a = qubits[2 * i], b = qubits[2 * i + 1];
        if (a < 0 || a >= s->n || (two && (b < 0 || b >= s->n)))
            return fail_code(QSV_ERR_INVALID, "gate " + std::to_string(i) +
                                                  " addresses a qubit outside the state");
        if (two && a == b)
            return fail_code(QSV_ERR_INVALID, "gate qubit indices must be distinct");
        if (!two && b != -1)
            return fail_code(QSV_ERR_INVALID, "one-qubit gate with a second qubit index");
    }
    return QSV_OK;
}

static int apply_gates_impl(qsv_state *s, int64_t n_gates, const int32_t *kinds,
                            const int32_t *qubits, const double *values, qsv_plan_stats *stats,
                            uint64_t basis);

int qsv_apply_gates(qsv_state *s, int64_t n_gates, const int32_t *kinds, const int32_t *qubits,
                    const double *values, qsv_plan_stats *stats)
{
    return apply_gates_impl(s, n_gates, kinds, qubits, values, stats, ~0ull);
}

int qsv_evolve_basis(qsv_state *s, uint64_t index, int64_t n_gates, const int32_t *kinds,
                     const int32_t *qubits, const double *values, qsv_plan_stats *stats)
{
    if (int rc = check_state(s)) return rc;
    if (index >= s->dim) return fail_code(QSV_ERR_INVALID, "basis index out of range");
    return apply_gates_impl(s, n_gates, kinds, qubits, values, stats, index);
}

// Small-state rotation programs (qsv_small.cu): on by default, QSV_SMALL=0
// runs them as tile passes (A/B and parity cross-checks).
static bool small_enabled()
{
    const char *e = getenv("QSV_SMALL");
    return !(e && e[0] == '0');
}

static int64_t g_small_launches = 0;

// The structure-only arrays of a small program live on the device once per
// (template, device); an evolve uploads only its angles.
static int small_dev_copy(const SmallProgram &sp, int device, const SmallProgram::DevCopy **out)
{
    for (const auto &d : sp.dev)
        if (d->device == device) {
            *out = d.get();
            return QSV_OK;
        }
    Blob b;
    auto d = std::make_shared<SmallProgram::DevCopy>();
    d->device = device;
    d->o_groups = b.add(sp.groups.data(), sp.groups.size() * sizeof(SmallGroup));
    d->o_meta = b.add(sp.meta.data(), sp.meta.size() * sizeof(int32_t));
    d->o_runs = b.add(sp.runs.data(), sp.runs.size() * sizeof(int32_t));
    d->o_xo = b.add(sp.xo.data(), sp.xo.size() * sizeof(uint32_t));
    d->o_tab = b.add(sp.tab.data(), sp.tab.size() * sizeof(uint32_t));
    if (cudaMalloc(&d->base, b.bytes.size()) != cudaSuccess) {
        cudaGetLastError();
        d->base = nullptr;
        return fail_code(QSV_ERR_NOMEM, "small-program tables: device allocation failed");
    }
    QSV_CUDA(cudaMemcpy(d->base, b.bytes.data(), b.bytes.size(), cudaMemcpyHostToDevice));
    sp.dev.push_back(d);
    *out = d.get();
    return QSV_OK;
}

static int run_small(qsv_state *s, const ProgramTemplate &t, const double *values, uint64_t basis)
{
    HostProfile prof("run_small");
    DeviceCtx *c = nullptr;
    if (int rc = ctx_for(s->device, &c)) return rc;
    const SmallProgram &sp = t.small;
    const SmallProgram::DevCopy *dc = nullptr;
    if (int rc = small_dev_copy(sp, s->device, &dc)) return rc;
    prof.mark("tables");
    // the angles go straight into the pinned staging buffer (one H2D copy)
    const size_t bytes = sp.src.size() * sizeof(double);
    if (int rc = ensure_work(*c, s->stream, bytes + 256)) return rc;
    if (int rc = ensure_stage(*c, bytes)) return rc;
    prof.mark("stage");
    double *th = reinterpret_cast<double *>(c->h_stage);
    uint64_t bad = 0;
    for (size_t r = 0; r < sp.src.size(); ++r) {
        th[r] = values[3 * (size_t)sp.src[r]];
        uint64_t bits;
        std::memcpy(&bits, th + r, 8);
        bad |= (uint64_t)(((bits >> 52) & 0x7ffu) == 0x7ffu);
    }
    if (bad) return fail_code(QSV_ERR_INVALID, "non-finite gate parameter");
    prof.mark("gather");
    QSV_CUDA(cudaMemcpyAsync(c->d_work, c->h_stage, bytes, cudaMemcpyHostToDevice, s->stream));
    QSV_CUDA(cudaEventRecord(c->stage_ev, s->stream));
    c->stage_pending = true;
    prof.mark("h2d");
    const char *k = dc->base;
    QSV_CUDA(launch_small(s->amps, s->n, basis, sp, (const SmallGroup *)(k + dc->o_groups),
                          (const int32_t *)(k + dc->o_meta), (const double *)c->d_work,
                          (const int32_t *)(k + dc->o_runs), (const uint32_t *)(k + dc->o_xo),
                          (const uint32_t *)(k + dc->o_tab), s->stream));
    prof.mark("launch");
    ++g_small_launches;
    return QSV_OK;
}

static int apply_gates_impl(qsv_state *s, int64_t n_gates, const int32_t *kinds,
                            const int32_t *qubits, const double *values, qsv_plan_stats *stats,
                            uint64_t basis)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(s)) return rc;
    if (n_gates < 0) return fail_code(QSV_ERR_INVALID, "negative gate count");
    if (n_gates == 0) {
        ProgramTemplate empty;
        fill_stats(empty, false, stats);
        if (basis != ~0ull) return qsv_set_basis(s, basis);
        return QSV_OK;
    }
    if (!kinds || !qubits || !values) return fail_code(QSV_ERR_INVALID, "null gate arrays");
    if (int rc = settle(s)) return rc;
    HostProfile prof("apply_gates");
    {
        // exponent all ones <=> inf / nan; an integer OR-reduction vectorises
        uint64_t bad = 0;
        for (int64_t i = 0; i < 3 * n_gates; ++i) {
            uint64_t b;
            std::memcpy(&b, values + i, 8);
            bad |= (uint64_t)(((b >> 52) & 0x7ffu) == 0x7ffu);
        }
        if (bad) return fail_code(QSV_ERR_INVALID, "non-finite gate parameter");
    }
    QSV_CUDA(cudaSetDevice(s->device));
    const uint64_t h = hash_structure(s->n, n_gates, kinds, qubits);
    const std::string knobs = planner_knobs();
    ProgramTemplate *tpl = nullptr;
    bool hit = false;
    for (auto it = g_cache.begin(); it != g_cache.end(); ++it) {
        if (it->hash == h && it->n == s->n && (int64_t)it->kinds.size() == n_gates &&
            it->knobs == knobs &&
            std::memcmp(it->kinds.data(), kinds, n_gates * 4) == 0 &&
            std::memcmp(it->qubits.data(), qubits, n_gates * 8) == 0) {
            g_cache.splice(g_cache.begin(), g_cache, it);
            tpl = &g_cache.front().tpl;
            ++g_cache.front().uses;
            hit = true;
            break;
        }
    }
    // a hit has the kinds / qubits of a structure validated when it was planned
    if (!tpl) {
        if (int rc = validate_gates(s, n_gates, kinds, qubits)) return rc;
        CacheEntry e;
        e.hash = h;
        e.n = s->n;
        e.knobs = knobs;
        e.kinds.assign(kinds, kinds + n_gates);
        e.qubits.assign(qubits, qubits + 2 * n_gates);
        plan_gates(s->n, n_gates, kinds, qubits, e.tpl);
        g_cache.push_front(std::move(e));
        if (g_cache.size() > kCacheMax) g_cache.pop_back();
        tpl = &g_cache.front().tpl;
    }
    prof.mark("lookup");
    if (tpl->small.valid && small_enabled()) {
        fill_stats(*tpl, hit, stats);
        return run_small(s, *tpl, values, basis);
    }
    if (!plain_u3() && needs_plain_u3(*tpl, values)) {
        // an angle the normalised U3 forms cannot take: a plan without them
        PlainU3Scope plain;
        return apply_gates_impl(s, n_gates, kinds, qubits, values, stats, basis);
    }
    CacheEntry &ce = g_cache.front();
    const bool dev_gmats = fast_path(s, *tpl, &ce.jc, ce.uses + 1) && !tpl->gfills.empty();
    std::vector<double> params(tpl->n_params);
    materialize_params(*tpl, values, params.data(), !dev_gmats);
    prof.mark("materialize");
    fill_stats(*tpl, hit, stats);
    const int rc = run_template(s, *tpl, params, ce.uses + 1, &ce.jc, dev_gmats, basis);
    prof.mark("run");
    return rc;
}

// Prepared programs (qsv_prepare_gates): a validated, planned structure
// addressed by id, so a caller that re-runs one circuit structure with new
// angles (a VQE loop) skips the per-call structure lookup.
static std::map<int64_t, CacheEntry> g_prepared;
static int64_t g_next_program = 1;

int qsv_prepare_gates(int n_qubits, int64_t n_gates, const int32_t *kinds, const int32_t *qubits,
                      int64_t *program_id)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!program_id) return fail_code(QSV_ERR_INVALID, "null output");
    *program_id = 0;
    if (n_qubits < 1 || n_qubits > kMaxQubits)
        return fail_code(QSV_ERR_RESOURCE, "qubit count out of range");
    if (n_gates < 0 || (n_gates > 0 && (!kinds || !qubits)))
        return fail_code(QSV_ERR_INVALID, "bad gate arrays");
    qsv_state fake;
    fake.n = n_qubits;
    if (int rc = validate_gates(&fake, n_gates, kinds, qubits)) return rc;
    CacheEntry e;
    e.hash = 0;
    e.n = n_qubits;
    // an identical structure already planned by qsv_apply_gates: copy its plan
    // (and its specialised modules) instead of planning again
    const uint64_t h = n_gates > 0 ? hash_structure(n_qubits, n_gates, kinds, qubits) : 0;
    bool copied = false;
    for (const CacheEntry &c : g_cache)
        if (n_gates > 0 && c.hash == h && c.n == n_qubits && (int64_t)c.kinds.size() == n_gates &&
            std::memcmp(c.kinds.data(), kinds, n_gates * 4) == 0 &&
            std::memcmp(c.qubits.data(), qubits, n_gates * 8) == 0) {
            e = c;
            copied = true;
            break;
        }
    if (!copied) {
        e.kinds.assign(kinds, kinds + n_gates);
        e.qubits.assign(qubits, qubits + 2 * n_gates);
        if (n_gates > 0) plan_gates(n_qubits, n_gates, kinds, qubits, e.tpl);
    }
    const int64_t id = g_next_program++;
    g_prepared.emplace(id, std::move(e));
    *program_id = id;
    return QSV_OK;
}

static int apply_prepared_impl(qsv_state *s, int64_t program_id, const double *values,
                               qsv_plan_stats *stats, uint64_t basis);

int qsv_apply_prepared(qsv_state *s, int64_t program_id, const double *values, qsv_plan_stats *stats)
{
    return apply_prepared_impl(s, program_id, values, stats, ~0ull);
}

int qsv_evolve_basis_prepared(qsv_state *s, uint64_t index, int64_t program_id, const double *values,
                              qsv_plan_stats *stats)
{
    if (int rc = check_state(s)) return rc;
    if (index >= s->dim) return fail_code(QSV_ERR_INVALID, "basis index out of range");
    return apply_prepared_impl(s, program_id, values, stats, index);
}

static int apply_prepared_impl(qsv_state *s, int64_t program_id, const double *values,
                               qsv_plan_stats *stats, uint64_t basis)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(s)) return rc;
    auto it = g_prepared.find(program_id);
    if (it == g_prepared.end()) return fail_code(QSV_ERR_INVALID, "unknown program id");
    CacheEntry &e = it->second;
    if (e.n != s->n) return fail_code(QSV_ERR_INVALID, "program and state qubit counts differ");
    const int64_t n_gates = (int64_t)e.kinds.size();
    if (n_gates == 0) {
        ProgramTemplate empty;
        fill_stats(empty, false, stats);
        if (basis != ~0ull) return qsv_set_basis(s, basis);
        return QSV_OK;
    }
    if (!values) return fail_code(QSV_ERR_INVALID, "null gate values");
    if (int rc = settle(s)) return rc;
    QSV_CUDA(cudaSetDevice(s->device));
    if (e.tpl.small.valid && small_enabled()) {
        // only the rotation angles are read (and checked) on this path
        fill_stats(e.tpl, e.uses++ > 0, stats);
        return run_small(s, e.tpl, values, basis);
    }
    uint64_t bad = 0;
    for (int64_t i = 0; i < 3 * n_gates; ++i) {
        uint64_t b;
        std::memcpy(&b, values + i, 8);
        bad |= (uint64_t)(((b >> 52) & 0x7ffu) == 0x7ffu);
    }
    if (bad) return fail_code(QSV_ERR_INVALID, "non-finite gate parameter");
    if (!plain_u3() && needs_plain_u3(e.tpl, values)) {
        PlainU3Scope plain;  // structure-cache path with a plan without normalised U3 forms
        return apply_gates_impl(s, n_gates, e.kinds.data(), e.qubits.data(), values, stats, basis);
    }
    const bool hit = e.uses > 0;
    ++e.uses;
    const bool dev_gmats = fast_path(s, e.tpl, &e.jc, e.uses) && !e.tpl.gfills.empty();
    std::vector<double> params(e.tpl.n_params);
    materialize_params(e.tpl, values, params.data(), !dev_gmats);
    fill_stats(e.tpl, hit, stats);
    return run_template(s, e.tpl, params, e.uses, &e.jc, dev_gmats, basis);
}

int qsv_release_program(int64_t program_id)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    g_prepared.erase(program_id);
    return QSV_OK;
}

static bool sweep_is_wide(const SweepPlan &sp)
{
    return !sp.groups.empty() && (sp.groups.front().pad[0] & 1);
}

static int validate_masks(int n, int64_t S, const uint64_t *x, const uint64_t *y,
                          const uint64_t *z)
{
    const uint64_t allowed = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
    for (int64_t t = 0; t < S; ++t) {
        if ((x[t] | y[t] | z[t]) & ~allowed)
            return fail_code(QSV_ERR_INVALID, "string index out of range for " + std::to_string(n) +
                                                  " qubits");
        if ((x[t] & y[t]) | (x[t] & z[t]) | (y[t] & z[t]))
            return fail_code(QSV_ERR_INVALID, "X/Y/Z masks of a string overlap");
    }
    return QSV_OK;
}

int qsv_apply_pauli_rotations(qsv_state *s, int64_t n, const uint64_t *x, const uint64_t *y,
                              const uint64_t *z, const double *theta, qsv_plan_stats *stats)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(s)) return rc;
    if (n < 0) return fail_code(QSV_ERR_INVALID, "negative rotation count");
    if (n == 0) return QSV_OK;
    if (!x || !y || !z || !theta) return fail_code(QSV_ERR_INVALID, "null rotation arrays");
    if (int rc = settle(s)) return rc;
    if (int rc = validate_masks(s->n, n, x, y, z)) return rc;
    for (int64_t r = 0; r < n; ++r)
        if (!std::isfinite(theta[r])) return fail_code(QSV_ERR_INVALID, "non-finite rotation angle");
    QSV_CUDA(cudaSetDevice(s->device));
    std::vector<Rot> R;
    R.reserve(n);
    for (int64_t r = 0; r < n; ++r) {
        if ((x[r] | y[r] | z[r]) == 0) continue;  // identity: global phase exp(-i t/2)
        R.push_back(Rot{x[r], y[r], z[r], (int)r});
    }
    ProgramTemplate t;
    plan_rotations(s->n, R, n, t);
    materialize_rotations(t, theta);
    std::vector<double> params(t.n_params);
    materialize_gmats(t, params.data());
    fill_stats(t, false, stats);
    int rc = run_template(s, t, params);
    if (rc) return rc;
    // identity strings contribute a global phase exp(-i theta/2)
    double ph_re = 1.0, ph_im = 0.0;
    bool any = false;
    for (int64_t r = 0; r < n; ++r) {
        if ((x[r] | y[r] | z[r]) != 0) continue;
        const double c = std::cos(0.5 * theta[r]), sn = -std::sin(0.5 * theta[r]);
        const double nr = ph_re * c - ph_im * sn, ni = ph_re * sn + ph_im * c;
        ph_re = nr;
        ph_im = ni;
        any = true;
    }
    if (any) QSV_CUDA(launch_axpby(s->amps, s->amps, s->dim, ph_re, ph_im, 0.0, 0.0, s->stream));
    return QSV_OK;
}

// States of <= 12 qubits: one warp per string (qsv_small.cu), no sweep plan;
// QSV_SMALL_EXPECT=0 takes the general sweeps (A/B and cross-checks).
static bool small_expect_enabled()
{
    const char *e = getenv("QSV_SMALL_EXPECT");
    return !(e && e[0] == '0');
}

static void finish_expectation(const std::vector<double> &vals, int64_t S, const double *coef_re,
                               const double *coef_im, double *out_re, double *out_im, double *per_term)
{
    // term-order accumulation, as statevector.py:104-107
    double re = 0.0, im = 0.0;
    for (int64_t t = 0; t < S; ++t) {
        re += coef_re[t] * vals[t];
        if (coef_im) im += coef_im[t] * vals[t];
    }
    *out_re = re;
    *out_im = im;
    if (per_term) std::memcpy(per_term, vals.data(), (size_t)S * 8);
}

// Device copies of small-state string records (flip, sign mask, ny mod 4),
// keyed by the masks: an energy loop re-evaluates the same Hamiltonian, so
// its records go up once (per device), not per call.
struct SmallExpEntry {
    uint64_t hash = 0;
    int device = -1, n = 0;
    std::vector<uint64_t> x, y, z;
    uint32_t *d_rec = nullptr;
};
static std::list<SmallExpEntry> g_small_exp;

static int small_exp_records(const qsv_state *s, int64_t S, const uint64_t *x, const uint64_t *y,
                             const uint64_t *z, const uint32_t **d_rec)
{
    const uint64_t h = hash_masks(s->n, S, x, y, z);
    for (auto it = g_small_exp.begin(); it != g_small_exp.end(); ++it)
        if (it->hash == h && it->device == s->device && it->n == s->n && (int64_t)it->x.size() == S &&
            std::memcmp(it->x.data(), x, S * 8) == 0 && std::memcmp(it->y.data(), y, S * 8) == 0 &&
            std::memcmp(it->z.data(), z, S * 8) == 0) {
            g_small_exp.splice(g_small_exp.begin(), g_small_exp, it);
            *d_rec = g_small_exp.front().d_rec;
            return QSV_OK;
        }
    std::vector<uint32_t> rec(4 * (size_t)S);
    for (int64_t t = 0; t < S; ++t) {
        rec[4 * t + 0] = (uint32_t)(x[t] | y[t]);
        rec[4 * t + 1] = (uint32_t)(y[t] | z[t]);
        rec[4 * t + 2] = (uint32_t)(__builtin_popcountll(y[t]) & 3);
        rec[4 * t + 3] = 0;
    }
    SmallExpEntry e;
    e.hash = h;
    e.device = s->device;
    e.n = s->n;
    e.x.assign(x, x + S);
    e.y.assign(y, y + S);
    e.z.assign(z, z + S);
    if (cudaMalloc((void **)&e.d_rec, rec.size() * 4) != cudaSuccess) {
        cudaGetLastError();
        return fail_code(QSV_ERR_NOMEM, "small expectation records: device allocation failed");
    }
    QSV_CUDA(cudaMemcpy(e.d_rec, rec.data(), rec.size() * 4, cudaMemcpyHostToDevice));
    g_small_exp.push_front(std::move(e));
    if (g_small_exp.size() > 8) {  // cudaFree synchronises the device: only on eviction
        SmallExpEntry &old = g_small_exp.back();
        cudaSetDevice(old.device);
        cudaFree(old.d_rec);
        cudaSetDevice(s->device);
        g_small_exp.pop_back();
    }
    *d_rec = g_small_exp.front().d_rec;
    return QSV_OK;
}

static int expectation_small(const qsv_state *s, DeviceCtx &c, int64_t S, const uint64_t *x, const uint64_t *y,
                             const uint64_t *z, const double *coef_re, const double *coef_im, double *out_re,
                             double *out_im, double *per_term, qsv_plan_stats *stats)
{
    HostProfile prof("expectation_small");
    const uint32_t *d_rec = nullptr;
    if (int rc = small_exp_records(s, S, x, y, z, &d_rec)) return rc;
    prof.mark("records");
    // the kernel writes the per-term values straight into the pinned staging
    // buffer (host memory the device addresses under UVA): no D2H copy call
    if (int rc = ensure_stage(c, (size_t)S * 8)) return rc;
    QSV_CUDA(launch_expect_small(s->amps, s->n, d_rec, (int)S, (double *)c.h_stage, num_sms(s->device),
                                 s->stream));
    prof.mark("launch");
    QSV_CUDA(cudaStreamSynchronize(s->stream));
    prof.mark("sync");
    std::vector<double> vals(S);
    std::memcpy(vals.data(), c.h_stage, (size_t)S * 8);
    finish_expectation(vals, S, coef_re, coef_im, out_re, out_im, per_term);
    qsv_plan_stats st{};
    st.n_input_ops = S;
    st.n_items = 1;
    st.n_passes = 1;
    st.tile_bits = s->n;
    st.cache_hit = 1;
    g_last_stats = st;
    if (stats) *stats = st;
    return QSV_OK;
}

int qsv_expectation(const qsv_state *s, int64_t S, const uint64_t *x, const uint64_t *y,
                    const uint64_t *z, const double *coef_re, const double *coef_im,
                    double *out_re, double *out_im, double *per_term, qsv_plan_stats *stats)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(s)) return rc;
    if (!out_re || !out_im) return fail_code(QSV_ERR_INVALID, "null outputs");
    *out_re = 0.0;
    *out_im = 0.0;
    if (S < 0) return fail_code(QSV_ERR_INVALID, "negative term count");
    if (S == 0) return QSV_OK;
    if (!x || !y || !z || !coef_re) return fail_code(QSV_ERR_INVALID, "null term arrays");
    if (int rc = validate_masks(s->n, S, x, y, z)) return rc;
    QSV_CUDA(cudaSetDevice(s->device));
    DeviceCtx *c = nullptr;
    if (int rc = ctx_for(s->device, &c)) return rc;
    if (s->n <= kSmallMaxQubits && small_expect_enabled())
        return expectation_small(s, *c, S, x, y, z, coef_re, coef_im, out_re, out_im, per_term, stats);

    HostProfile prof("expectation");
    const uint64_t h = hash_masks(s->n, S, x, y, z);
    const bool jit = jit_enabled(s->n);
    const std::string knobs = planner_knobs();
    std::vector<SweepPlan> *plan = nullptr;
    std::vector<std::string> *jsrc = nullptr;
    bool hit = false;
    for (auto it = g_exp_cache.begin(); it != g_exp_cache.end(); ++it) {
        if (it->hash == h && it->n == s->n && it->jit == jit && (int64_t)it->x.size() == S &&
            it->knobs == knobs &&
            std::memcmp(it->x.data(), x, S * 8) == 0 && std::memcmp(it->y.data(), y, S * 8) == 0 &&
            std::memcmp(it->z.data(), z, S * 8) == 0) {
            g_exp_cache.splice(g_exp_cache.begin(), g_exp_cache, it);
            plan = &g_exp_cache.front().plan;
            jsrc = &g_exp_cache.front().jit_src;
            hit = true;
            break;
        }
    }
    if (!plan) {
        ExpCacheEntry e;
        e.hash = h;
        e.n = s->n;
        e.knobs = knobs;
        e.x.assign(x, x + S);
        e.y.assign(y, y + S);
        e.z.assign(z, z + S);
        e.jit = jit;
        plan_expectation(s->n, S, x, y, z, e.plan, jit);
        e.jit_src.resize(e.plan.size());
        if (jit)
            for (size_t k = 0; k < e.plan.size(); ++k) jit_sweep_source(e.plan[k], e.jit_src[k]);
        g_exp_cache.push_front(std::move(e));
        if (g_exp_cache.size() > 4) g_exp_cache.pop_back();
        plan = &g_exp_cache.front().plan;
        jsrc = &g_exp_cache.front().jit_src;
    }
    if (jit) {
        std::vector<const std::string *> srcs;
        for (const std::string &src : *jsrc)
            if (!src.empty()) srcs.push_back(&src);
        std::string err;
        if (!srcs.empty() && jit_prepare(s->device, srcs, err) && getenv("QSV_JIT_VERBOSE"))
            fprintf(stderr, "qsv jit: %s\n", err.c_str());
    }
    prof.mark("plan");
    // blob: per sweep groups / terms / map / gflip
    Blob b;
    struct Off { size_t g, t, m, f, off, comp; int rows; };
    std::vector<Off> offs;
    size_t max_partial = 0;
    for (const SweepPlan &sp : *plan) {
        Off o;
        o.g = b.add(sp.groups.data(), sp.groups.size() * sizeof(GroupRec));
        o.t = b.add(sp.terms.data(), sp.terms.size() * sizeof(TermRec));
        o.m = b.add(sp.map.data(), sp.map.size() * sizeof(int32_t));
        o.f = b.add(sp.gflip.data(), sp.gflip.size() * sizeof(uint64_t));
        o.off = o.comp = 0;
        if (!sp.global) {
            std::vector<uint64_t> offhi;
            std::vector<int32_t> comp;
            geom_tables(sp.geom, offhi, comp);
            o.off = b.add(offhi.data(), offhi.size() * sizeof(uint64_t));
            o.comp = b.add(comp.data(), comp.size() * sizeof(int32_t));
        }
        o.rows = sp.global ? expect_global_grid(s->n)
                           : expect_sweep_grid(dims_of(sp.geom), (int)sp.terms.size(), sp.ndiag,
                                             (int)sp.groups.size(), sweep_is_wide(sp));
        max_partial = std::max(max_partial, (size_t)std::max(o.rows, 16 * num_sms(s->device)) *
                                                sp.terms.size());
        offs.push_back(o);
    }
    const size_t per_term_bytes = ((size_t)S * 8 + 255) & ~(size_t)255;
    char *d = nullptr;
    size_t scratch = 0;
    if (int rc = upload_blob(*c, s->stream, b, per_term_bytes + max_partial * 8 + 256, &d, &scratch))
        return rc;
    double *d_per_term = (double *)(d + scratch);
    double *d_partial = (double *)(d + scratch + per_term_bytes);
    prof.mark("upload");
    for (size_t k = 0; k < plan->size(); ++k) {
        const SweepPlan &sp = (*plan)[k];
        const Off &o = offs[k];
        const int nterms = (int)sp.terms.size();
        if (nterms == 0) continue;
        int rows = 0;
        if (sp.global) {
            QSV_CUDA(launch_expect_global(s->amps, s->n, (const GroupRec *)(d + o.g),
                                          (const uint64_t *)(d + o.f), (int)sp.groups.size(),
                                          (const TermRec *)(d + o.t), nterms, d_partial, &rows,
                                          s->stream));
        } else if (jit && !(*jsrc)[k].empty() &&
                   jit_sweep_launch(s->device, (*jsrc)[k], s->amps, dims_of(sp.geom),
                                    (const uint64_t *)(d + o.off), (const int32_t *)(d + o.comp),
                                    d_partial,
                                    (int)std::min<uint64_t>(1ull << sp.geom.ncomp,
                                                            (uint64_t)num_sms(s->device)),
                                    s->stream)) {
            rows = 16 * (int)std::min<uint64_t>(1ull << sp.geom.ncomp, (uint64_t)num_sms(s->device));
            ++g_jit_launches;
        } else {
            QSV_CUDA(launch_expect_sweep(s->amps, dims_of(sp.geom), (const uint64_t *)(d + o.off),
                                         (const int32_t *)(d + o.comp), (const GroupRec *)(d + o.g),
                                         (int)sp.groups.size(), (const TermRec *)(d + o.t), nterms,
                                         sp.ndiag, sweep_is_wide(sp), d_partial, &rows, s->stream));
        }
        QSV_CUDA(launch_reduce_columns(d_partial, rows, nterms, (const int32_t *)(d + o.m),
                                       d_per_term, s->stream));
    }
    prof.mark("launches");
    std::vector<double> vals(S);
    if (int rc = ensure_stage(*c, (size_t)S * 8)) return rc;
    QSV_CUDA(cudaMemcpyAsync(c->h_stage, d_per_term, (size_t)S * 8, cudaMemcpyDeviceToHost, s->stream));
    QSV_CUDA(cudaStreamSynchronize(s->stream));
    prof.mark("sync");
    std::memcpy(vals.data(), c->h_stage, (size_t)S * 8);
    finish_expectation(vals, S, coef_re, coef_im, out_re, out_im, per_term);
    qsv_plan_stats st{};
    st.n_input_ops = S;
    st.n_items = (int64_t)plan->size();
    st.n_passes = (int64_t)plan->size();
    for (const SweepPlan &sp : *plan) st.n_fallback += sp.global ? 1 : 0;
    st.tile_bits = plan->empty() ? 0 : plan->front().geom.m;
    st.cache_hit = hit ? 1 : 0;
    g_last_stats = st;
    if (stats) *stats = st;
    return QSV_OK;
}

int qsv_apply_pauli(const qsv_state *src, qsv_state *dst, uint64_t x, uint64_t y, uint64_t z)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(src)) return rc;
    if (int rc = check_state(dst)) return rc;
    if (src->n != dst->n) return fail_code(QSV_ERR_INVALID, "state qubit counts differ");
    if (src == dst) return fail_code(QSV_ERR_INVALID, "apply_pauli needs distinct src and dst");
    if (int rc = validate_masks(src->n, 1, &x, &y, &z)) return rc;
    QSV_CUDA(cudaSetDevice(src->device));
    if (int rc = settle(dst, dst->stream != src->stream)) return rc;
    QSV_CUDA(launch_apply_pauli(src->amps, dst->amps, src->dim, x, y, z, 1.0, 0.0, 0, src->stream));
    return QSV_OK;
}

int qsv_apply_operator(const qsv_state *src, qsv_state *dst, int64_t S, const uint64_t *x,
                       const uint64_t *y, const uint64_t *z, const double *coef_re,
                       const double *coef_im)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(src)) return rc;
    if (int rc = check_state(dst)) return rc;
    if (src->n != dst->n) return fail_code(QSV_ERR_INVALID, "state qubit counts differ");
    if (src == dst) return fail_code(QSV_ERR_INVALID, "apply_operator needs distinct src and dst");
    if (S < 0 || (S > 0 && (!x || !y || !z || !coef_re)))
        return fail_code(QSV_ERR_INVALID, "bad term arrays");
    if (int rc = validate_masks(src->n, S, x, y, z)) return rc;
    QSV_CUDA(cudaSetDevice(src->device));
    if (int rc = settle(dst, dst->stream != src->stream)) return rc;
    if (S == 0) {
        QSV_CUDA(cudaMemsetAsync(dst->amps, 0, 16 * dst->dim, src->stream));
        return QSV_OK;
    }
    if (src->n <= 16 && S >= 4) {
        // small (L2-resident) state: one kernel over all strings instead of S
        // launches, same per-string arithmetic and order
        DeviceCtx *c = nullptr;
        if (int rc = ctx_for(src->device, &c)) return rc;
        std::vector<uint64_t> fs(2 * S);
        std::vector<double> cf(2 * S);
        for (int64_t t = 0; t < S; ++t) {
            fs[2 * t] = x[t] | y[t];
            fs[2 * t + 1] = y[t] | z[t];
            const int wy = __builtin_popcountll(y[t]) & 3;  // i^{|y|}, as launch_apply_pauli
            double pre = 1.0, pim = 0.0;
            if (wy == 1) { pre = 0.0; pim = 1.0; }
            else if (wy == 2) { pre = -1.0; }
            else if (wy == 3) { pre = 0.0; pim = -1.0; }
            const double cre = coef_re[t], cim = coef_im ? coef_im[t] : 0.0;
            cf[2 * t] = cre * pre - cim * pim;
            cf[2 * t + 1] = cre * pim + cim * pre;
        }
        Blob b;
        const size_t of = b.add(fs.data(), fs.size() * 8), oc = b.add(cf.data(), cf.size() * 8);
        char *d = nullptr;
        size_t scratch = 0;
        if (int rc = upload_blob(*c, src->stream, b, 0, &d, &scratch)) return rc;
        QSV_CUDA(launch_apply_operator_small(src->amps, dst->amps, src->dim, (const uint64_t *)(d + of),
                                             (const double2 *)(d + oc), (int)S, src->stream));
        return QSV_OK;
    }
    for (int64_t t = 0; t < S; ++t) {
        QSV_CUDA(launch_apply_pauli(src->amps, dst->amps, src->dim, x[t], y[t], z[t], coef_re[t],
                                    coef_im ? coef_im[t] : 0.0, t > 0 ? 1 : 0, src->stream));
    }
    return QSV_OK;
}

static int dot_common(const qsv_state *a, const qsv_state *b, int mode, double *out2)
{
    DeviceCtx *c = nullptr;
    if (int rc = ctx_for(a->device, &c)) return rc;
    const size_t part = (size_t)num_sms(a->device) * 4 * 2 * sizeof(double);
    if (int rc = ensure_work(*c, a->stream, part + 256)) return rc;
    double *d_part = (double *)c->d_work;
    double *d_out = (double *)((char *)c->d_work + ((part + 255) & ~(size_t)255));
    QSV_CUDA(launch_dot(a->amps, b ? b->amps : nullptr, a->dim, d_part, d_out, mode, a->stream));
    if (int rc = ensure_stage(*c, 16)) return rc;
    QSV_CUDA(cudaMemcpyAsync(c->h_stage, d_out, 16, cudaMemcpyDeviceToHost, a->stream));
    QSV_CUDA(cudaStreamSynchronize(a->stream));
    std::memcpy(out2, c->h_stage, 16);
    return QSV_OK;
}

int qsv_vdot(const qsv_state *a, const qsv_state *b, double *out2)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(a)) return rc;
    if (int rc = check_state(b)) return rc;
    if (!out2) return fail_code(QSV_ERR_INVALID, "null output");
    if (a->n != b->n) return fail_code(QSV_ERR_INVALID, "state qubit counts differ");
    QSV_CUDA(cudaSetDevice(a->device));
    return dot_common(a, b, 0, out2);
}

int qsv_norm(const qsv_state *s, double *out)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(s)) return rc;
    if (!out) return fail_code(QSV_ERR_INVALID, "null output");
    QSV_CUDA(cudaSetDevice(s->device));
    double v[2];
    if (int rc = dot_common(s, nullptr, 1, v)) return rc;
    *out = std::sqrt(v[0]);
    return QSV_OK;
}

int qsv_rotation_adjoint(qsv_state *phi, qsv_state *lam, int64_t R, const uint64_t *x,
                         const uint64_t *y, const uint64_t *z, const double *theta, double *grad)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(phi)) return rc;
    if (int rc = check_state(lam)) return rc;
    if (phi == lam) return fail_code(QSV_ERR_INVALID, "rotation_adjoint needs distinct states");
    if (phi->n != lam->n) return fail_code(QSV_ERR_INVALID, "state qubit counts differ");
    if (R < 0) return fail_code(QSV_ERR_INVALID, "negative rotation count");
    if (R == 0) return QSV_OK;
    if (!x || !y || !z || !theta || !grad) return fail_code(QSV_ERR_INVALID, "null arrays");
    if (int rc = validate_masks(phi->n, R, x, y, z)) return rc;
    for (int64_t r = 0; r < R; ++r)
        if (!std::isfinite(theta[r])) return fail_code(QSV_ERR_INVALID, "non-finite rotation angle");
    QSV_CUDA(cudaSetDevice(phi->device));
    if (int rc = settle(phi)) return rc;
    if (int rc = settle(lam, lam->stream != phi->stream)) return rc;
    if (lam->stream != phi->stream) QSV_CUDA(cudaStreamSynchronize(lam->stream));
    DeviceCtx *c = nullptr;
    if (int rc = ctx_for(phi->device, &c)) return rc;
    std::vector<double> cs(2 * R);  // cos, sin of theta/2 (as the rotation passes: host libm)
    for (int64_t r = 0; r < R; ++r) {
        cs[2 * r] = std::cos(0.5 * theta[r]);
        cs[2 * r + 1] = std::sin(0.5 * theta[r]);
    }
    Blob b;
    const size_t ox = b.add(x, R * 8), oy = b.add(y, R * 8), oz = b.add(z, R * 8),
                 ot = b.add(cs.data(), R * 16);
    const size_t scratch_doubles = adjoint_scratch_doubles(phi->n, R, phi->device);
    char *d = nullptr;
    size_t scratch = 0;
    if (int rc = upload_blob(*c, phi->stream, b, (scratch_doubles + R) * 8 + 256, &d, &scratch))
        return rc;
    double *d_grad = (double *)(d + scratch);
    double *d_scr = d_grad + R;
    QSV_CUDA(launch_rotation_adjoint(phi->amps, lam->amps, phi->n, R, (const uint64_t *)(d + ox),
                                     (const uint64_t *)(d + oy), (const uint64_t *)(d + oz), x, y, z,
                                     (const double2 *)(d + ot), d_scr, d_grad, phi->stream));
    if (int rc = ensure_stage(*c, (size_t)R * 8)) return rc;
    QSV_CUDA(cudaMemcpyAsync(c->h_stage, d_grad, (size_t)R * 8, cudaMemcpyDeviceToHost, phi->stream));
    QSV_CUDA(cudaStreamSynchronize(phi->stream));
    std::memcpy(grad, c->h_stage, (size_t)R * 8);
    return QSV_OK;
}

int qsv_axpby(qsv_state *y, const qsv_state *x, double are, double aim, double bre, double bim)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(y)) return rc;
    if (int rc = check_state(x)) return rc;
    if (x->n != y->n) return fail_code(QSV_ERR_INVALID, "state qubit counts differ");
    QSV_CUDA(cudaSetDevice(y->device));
    if (int rc = settle(y)) return rc;
    QSV_CUDA(launch_axpby(y->amps, x->amps, y->dim, are, aim, bre, bim, y->stream));
    return QSV_OK;
}

int qsv_apply_1q(qsv_state *s, const double *m, int qubit)
{
    if (int rc = check_state(s)) return rc;
    if (!m) return fail_code(QSV_ERR_INVALID, "null matrix");
    if (qubit < 0 || qubit >= s->n) return fail_code(QSV_ERR_INVALID, "qubit out of range");
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    QSV_CUDA(cudaSetDevice(s->device));
    if (int rc = settle(s)) return rc;
    ProgramTemplate t;
    int32_t kind = K_U3, q[2] = {qubit, -1};
    plan_gates(s->n, 1, &kind, q, t);
    for (OpRec &op : t.ops)
        if (op.type == OP_U1) op.h = 0;  // arbitrary caller matrix: general class
    // plan for a U3 gate: one OP_U1 whose params are the supplied matrix
    std::vector<double> params(t.n_params);
    std::memcpy(params.data(), m, 8 * sizeof(double));
    fill_stats(t, false, nullptr);
    return run_template(s, t, params);
}

int qsv_apply_2q(qsv_state *s, const double *m, int q0, int q1)
{
    if (int rc = check_state(s)) return rc;
    if (!m) return fail_code(QSV_ERR_INVALID, "null matrix");
    if (q0 < 0 || q0 >= s->n || q1 < 0 || q1 >= s->n || q0 == q1)
        return fail_code(QSV_ERR_INVALID, "bad qubit pair");
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    QSV_CUDA(cudaSetDevice(s->device));
    if (int rc = settle(s)) return rc;
    ProgramTemplate t;
    int32_t kind = K_CU3, q[2] = {q0, q1};
    plan_gates(s->n, 1, &kind, q, t);
    std::vector<double> params(t.n_params);
    std::memcpy(params.data(), m, 32 * sizeof(double));
    fill_stats(t, false, nullptr);
    return run_template(s, t, params);
}

int qsv_apply_matrix(qsv_state *s, int k, const int32_t *qubits, const double *m)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(s)) return rc;
    if (!m || !qubits) return fail_code(QSV_ERR_INVALID, "null matrix or qubit list");
    if (k < 1) return fail_code(QSV_ERR_INVALID, "k must be >= 1");
    if (k > 5 || k > s->n) return fail_code(QSV_ERR_RESOURCE, "dense blocks are limited to 5 qubits");
    uint64_t seen = 0;
    for (int i = 0; i < k; ++i) {
        if (qubits[i] < 0 || qubits[i] >= s->n) return fail_code(QSV_ERR_INVALID, "qubit out of range");
        if ((seen >> qubits[i]) & 1ull) return fail_code(QSV_ERR_INVALID, "duplicate qubit");
        seen |= 1ull << qubits[i];
    }
    QSV_CUDA(cudaSetDevice(s->device));
    if (int rc = settle(s)) return rc;
    DeviceCtx *c = nullptr;
    if (int rc = ctx_for(s->device, &c)) return rc;
    const size_t mb = (size_t)16 << (2 * k);
    Blob b;
    b.add(m, mb);
    char *d = nullptr;
    size_t scratch = 0;
    if (int rc = upload_blob(*c, s->stream, b, 0, &d, &scratch)) return rc;
    QSV_CUDA(launch_dense(s->amps, s->n, k, qubits, (const double2 *)d, num_sms(s->device), s->stream));
    return QSV_OK;
}

int qsv_match_rotations(int n, int64_t n_gates, const int32_t *kinds, const int32_t *qubits,
                        int64_t cap, int64_t *spans, uint64_t *masks, int64_t *count)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!count) return fail_code(QSV_ERR_INVALID, "null output");
    if (n < 1 || n > kMaxQubits) return fail_code(QSV_ERR_RESOURCE, "qubit count out of range");
    if (n_gates < 0 || (n_gates > 0 && (!kinds || !qubits)))
        return fail_code(QSV_ERR_INVALID, "bad gate arrays");
    qsv_state fake;
    fake.n = n;
    if (int rc = validate_gates(&fake, n_gates, kinds, qubits)) return rc;
    std::vector<RotSpan> out;
    match_rotations(n_gates, kinds, qubits, out);
    *count = (int64_t)out.size();
    for (int64_t k = 0; k < (int64_t)out.size() && k < cap; ++k) {
        if (spans) {
            spans[3 * k] = out[k].start;
            spans[3 * k + 1] = out[k].len;
            spans[3 * k + 2] = out[k].rz;
        }
        if (masks) {
            masks[3 * k] = out[k].x;
            masks[3 * k + 1] = out[k].y;
            masks[3 * k + 2] = out[k].z;
        }
    }
    return QSV_OK;
}

int qsv_plan_gates(int n, int64_t n_gates, const int32_t *kinds, const int32_t *qubits,
                   qsv_plan_stats *out)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!out) return fail_code(QSV_ERR_INVALID, "null output");
    if (n < 1 || n > kMaxQubits) return fail_code(QSV_ERR_RESOURCE, "qubit count out of range");
    if (n_gates < 0 || (n_gates > 0 && (!kinds || !qubits)))
        return fail_code(QSV_ERR_INVALID, "bad gate arrays");
    qsv_state fake;
    fake.n = n;
    if (int rc = validate_gates(&fake, n_gates, kinds, qubits)) return rc;
    ProgramTemplate t;
    plan_gates(n, n_gates, kinds, qubits, t);
    fill_stats(t, false, out);
    return QSV_OK;
}

int qsv_plan_expectation(int n, int64_t S, const uint64_t *x, const uint64_t *y,
                         const uint64_t *z, qsv_plan_stats *out)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!out) return fail_code(QSV_ERR_INVALID, "null output");
    if (n < 1 || n > kMaxQubits) return fail_code(QSV_ERR_RESOURCE, "qubit count out of range");
    if (S < 0 || (S > 0 && (!x || !y || !z))) return fail_code(QSV_ERR_INVALID, "bad term arrays");
    if (int rc = validate_masks(n, S, x, y, z)) return rc;
    std::vector<SweepPlan> plan;
    plan_expectation(n, S, x, y, z, plan);
    qsv_plan_stats st{};
    st.n_input_ops = S;
    st.n_items = (int64_t)plan.size();
    st.n_passes = (int64_t)plan.size();
    for (const SweepPlan &sp : plan) st.n_fallback += sp.global ? 1 : 0;
    st.tile_bits = plan.empty() ? 0 : plan.front().geom.m;
    *out = st;
    return QSV_OK;
}

int qsv_debug_pass_source(int n, int64_t n_gates, const int32_t *kinds, const int32_t *qubits,
                          int64_t k, char *out, int64_t cap, int64_t *needed, int64_t *n_passes)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (n < 1 || n > kMaxQubits) return fail_code(QSV_ERR_RESOURCE, "qubit count out of range");
    if (n_gates < 0 || (n_gates > 0 && (!kinds || !qubits))) return fail_code(QSV_ERR_INVALID, "bad gate arrays");
    qsv_state fake;
    fake.n = n;
    if (int rc = validate_gates(&fake, n_gates, kinds, qubits)) return rc;
    ProgramTemplate t;
    plan_gates(n, n_gates, kinds, qubits, t);
    if (n_passes) *n_passes = (int64_t)t.passes.size();
    std::string src;
    std::vector<OpRec> lops;
    std::vector<BlockRec> lblk;
    int r_lo, r_hi, p_lo, p_hi;
    if (k >= 0 && k < (int64_t)t.passes.size() && pass_local(t, (size_t)k, lops, lblk, r_lo, r_hi, p_lo, p_hi))
        jit_source(t.passes[k].geom, lblk.data(), (int)lblk.size(), lops.data(), t.rots.data() + r_lo,
                   p_hi - p_lo, src);
    if (needed) *needed = (int64_t)src.size() + 1;
    if (out && cap > (int64_t)src.size()) std::memcpy(out, src.c_str(), src.size() + 1);
    return QSV_OK;
}

int qsv_debug_sweep_source(int n, int64_t S, const uint64_t *x, const uint64_t *y,
                           const uint64_t *z, int64_t k, char *out, int64_t cap, int64_t *needed,
                           int64_t *n_sweeps)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (n < 1 || n > kMaxQubits) return fail_code(QSV_ERR_RESOURCE, "qubit count out of range");
    if (S < 0 || (S > 0 && (!x || !y || !z))) return fail_code(QSV_ERR_INVALID, "bad term arrays");
    if (int rc = validate_masks(n, S, x, y, z)) return rc;
    std::vector<SweepPlan> plan;
    plan_expectation(n, S, x, y, z, plan, true);
    if (n_sweeps) *n_sweeps = (int64_t)plan.size();
    std::string src;
    if (k >= 0 && k < (int64_t)plan.size()) jit_sweep_source(plan[k], src);
    if (needed) *needed = (int64_t)src.size() + 1;
    if (out && cap > (int64_t)src.size()) std::memcpy(out, src.c_str(), src.size() + 1);
    return QSV_OK;
}

// Debug export of the compiled tile program (JSON) for the CPU emulator in
// tests/ -- lets the planner and its encoding be verified without a GPU.
int qsv_debug_plan_json(int n, int64_t n_gates, const int32_t *kinds, const int32_t *qubits,
                        const double *values, char *out, int64_t cap, int64_t *needed)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (n < 1 || n > kMaxQubits) return fail_code(QSV_ERR_RESOURCE, "qubit count out of range");
    qsv_state fake;
    fake.n = n;
    if (int rc = validate_gates(&fake, n_gates, kinds, qubits)) return rc;
    ProgramTemplate t;
    plan_gates(n, n_gates, kinds, qubits, t);
    if (!plain_u3() && values && needs_plain_u3(t, values)) {  // as apply_gates_impl
        PlainU3Scope plain;
        return qsv_debug_plan_json(n, n_gates, kinds, qubits, values, out, cap, needed);
    }
    std::vector<double> params(t.n_params);
    materialize_params(t, values, params.data());
    std::string j = "{\"n\":" + std::to_string(n) + ",\"block_bits\":" + std::to_string(kBlockBits);
    // the small-state rotation program (qsv_small.cu), when the plan has one
    j += ",\"small\":{\"valid\":" + std::to_string(t.small.valid ? 1 : 0) + ",\"ncls\":" +
         std::to_string(t.small.ncls) + ",\"share\":" + std::to_string(t.small.share) + ",\"w\":[" +
         std::to_string(t.small.w[0]) + "," + std::to_string(t.small.w[1]) + "," + std::to_string(t.small.w[2]) +
         "],\"groups\":[";
    // [xm, r0, r1, dimb, h, pm0..3, lu0, lu1]
    for (size_t g = 0; g < t.small.groups.size(); ++g) {
        const SmallGroup &G = t.small.groups[g];
        std::vector<int64_t> f = {G.xm, G.r0, G.r1, G.dimb, G.h, G.pm[0], G.pm[1], G.pm[2], G.pm[3], G.lu[0], G.lu[1]};
        j += g ? ",[" : "[";
        for (size_t i = 0; i < f.size(); ++i) j += (i ? "," : "") + std::to_string(f[i]);
        j += "]";
    }
    // the per-thread table and slot constants (small programs only: tests)
    j += "],\"nthr\":" + std::to_string(t.small.nthr) + ",\"swz\":[" + std::to_string(t.small.swz[0]) + "," +
         std::to_string(t.small.swz[1]) + "," + std::to_string(t.small.swz[2]) + "],\"xo\":[";
    const bool emit_tab = t.small.tab.size() <= ((size_t)1 << 18);
    for (size_t i = 0; emit_tab && i < t.small.xo.size(); ++i) j += (i ? "," : "") + std::to_string(t.small.xo[i]);
    j += "],\"tab\":[";
    for (size_t i = 0; emit_tab && i < t.small.tab.size(); ++i)
        j += (i ? "," : "") + std::to_string(t.small.tab[i]);
    j += "],\"runs\":[";
    for (size_t i = 0; i < t.small.runs.size(); ++i) j += (i ? "," : "") + std::to_string(t.small.runs[i]);
    j += "]},\"passes\":[";
    char buf[256];
    for (size_t k = 0; k < t.passes.size(); ++k) {
        const PassPlan &p = t.passes[k];
        if (k) j += ",";
        j += "{\"global\":" + std::to_string(p.global ? 1 : 0);
        snprintf(buf, sizeof(buf), ",\"flip\":%llu", (unsigned long long)p.flip);
        j += buf;
        j += ",\"m\":" + std::to_string(p.geom.m) + ",\"c\":" + std::to_string(p.geom.c);
        j += ",\"pos\":[";
        for (int i = 0; i < p.geom.m; ++i) j += (i ? "," : "") + std::to_string(p.geom.pos[i]);
        j += "],\"comp\":[";
        for (int i = 0; i < p.geom.ncomp; ++i) j += (i ? "," : "") + std::to_string(p.geom.comp[i]);
        j += "],\"store_cols\":[";
        for (int i = 0; i < 12; ++i) j += (i ? "," : "") + std::to_string(p.store_cols[i]);
        j += "],\"store_t\":" + std::to_string(p.store_t);
        j += ",\"op_begin\":" + std::to_string(p.op_begin) + ",\"op_end\":" + std::to_string(p.op_end);
        j += ",\"blocks\":[";
        for (int b = p.block_begin; b < p.block_end; ++b) {
            const BlockRec &br = t.blocks[b];
            if (b > p.block_begin) j += ",";
            j += "{\"kind\":" + std::to_string(br.kind) + ",\"flags\":" + std::to_string(br.pad0) +
                 ",\"op0\":" + std::to_string(br.op0) +
                 ",\"op1\":" + std::to_string(br.op1) + ",\"tswz\":" + std::to_string(br.tswz) +
                 ",\"cols\":[";
            for (int i = 0; i < 12; ++i) j += (i ? "," : "") + std::to_string(br.cols[i]);
            j += "]}";
        }
        j += "]}";
    }
    j += "],\"ops\":[";
    for (size_t k = 0; k < t.ops.size(); ++k) {
        const OpRec &o = t.ops[k];
        snprintf(buf, sizeof(buf), "%s[%d,%d,%d,%d,%d,%d,%d,%u]", k ? "," : "", o.type, o.a, o.b, o.h,
                 o.r0, o.r1, o.p, o.f);
        j += buf;
    }
    j += "],\"rots\":[";
    for (size_t k = 0; k < t.rots.size(); ++k) {
        const RotRec &r = t.rots[k];
        snprintf(buf, sizeof(buf), "%s[%llu,%u,%d,%.17g,%.17g]", k ? "," : "",
                 (unsigned long long)r.s_hi, r.s_loc, r.q, r.c, r.s);
        j += buf;
    }
    j += "],\"params\":[";
    for (size_t k = 0; k < params.size(); ++k) {
        snprintf(buf, sizeof(buf), "%s%.17g", k ? "," : "", params[k]);
        j += buf;
    }
    j += "]}";
    if (needed) *needed = (int64_t)j.size() + 1;
    if (out && cap > (int64_t)j.size()) std::memcpy(out, j.c_str(), j.size() + 1);
    return QSV_OK;
}

int qsv_sample_parity(const qsv_state *s, uint64_t support_mask, int64_t shots,
                      const uint64_t *philox_key, double *out_mean, int64_t *outcomes)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (int rc = check_state(s)) return rc;
    if (!philox_key || !out_mean) return fail_code(QSV_ERR_INVALID, "null key or output");
    if (shots < 1) return fail_code(QSV_ERR_INVALID, "shots must be >= 1");
    if (s->n < 64 && (support_mask >> s->n)) return fail_code(QSV_ERR_INVALID, "support mask out of range");
    QSV_CUDA(cudaSetDevice(s->device));
    DeviceCtx *c = nullptr;
    if (int rc = ctx_for(s->device, &c)) return rc;
    const size_t scratch = sample_scratch_bytes(s->dim);
    const size_t out_bytes = outcomes ? (((size_t)shots * 8 + 255) & ~(size_t)255) : 0;
    if (int rc = ensure_work(*c, s->stream, scratch + out_bytes + 256)) return rc;
    if (c->stage_pending) {  // the workspace head may still feed an earlier program upload
        QSV_CUDA(cudaStreamSynchronize(s->stream));
        c->stage_pending = false;
    }
    int64_t *d_out = outcomes ? (int64_t *)((char *)c->d_work + scratch) : nullptr;
    unsigned long long odd = 0;
    QSV_CUDA(launch_sample_parity(s->amps, s->dim, shots, philox_key[0], philox_key[1], support_mask,
                                  c->d_work, scratch, d_out, &odd, s->stream));
    if (outcomes)
        QSV_CUDA(cudaMemcpy(outcomes, d_out, (size_t)shots * 8, cudaMemcpyDeviceToHost));
    // np.mean(1 - 2 parity): an exact integer sum, one rounding
    *out_mean = (double)(shots - 2 * (int64_t)odd) / (double)shots;
    return release_big_work(*c, s->stream);
}

int qsv_small_info(int64_t *launches)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (!launches) return fail_code(QSV_ERR_INVALID, "null output");
    *launches = g_small_launches;
    return QSV_OK;
}

int qsv_jit_info(int *available, int64_t *launches)
{
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    if (available) *available = jit_enabled(64) ? 1 : 0;
    if (launches) *launches = g_jit_launches;
    return QSV_OK;
}

int qsv_last_plan_stats(qsv_plan_stats *out)
{
    if (!out) return fail_code(QSV_ERR_INVALID, "null output");
    *out = g_last_stats;
    return QSV_OK;
}

}  // extern "C"
