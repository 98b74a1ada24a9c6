// qsv_planner.h -- host-side (native C++) fusion planner of the engine.
//
// Turns a bound gate list (the reference's Circuit, circuit.py:48-156) into a
// short sequence of HBM passes:
//   1. recognise pauli_evolution blocks (circuit.py:271-281: basis layer,
//      CNOT ladder, RZ, mirror) and replace each by one direct Pauli rotation
//      exp(-i theta/2 P) (theta = the RZ's bound value);
//   2. group consecutive rotations that share a flip mask (they act on the
//      same amplitude pairs, so one register sweep applies all of them);
//   3. schedule gates / rotation groups into shared-memory tile passes by a
//      dependency-aware first-fit: an item may move into an earlier pass past
//      anything it commutes with (disjoint qubits for gates, even symplectic
//      product for Pauli rotations), and a pass accepts it if its tile (low
//      contiguous bits + up to m - c other qubits) covers the qubits the item
//      must see (gate qubits / rotation flip bits; Z bits outside the tile are
//      a per-tile sign).
// Structural plans are cached by a hash of (n, kinds, qubits) so repeated
// energy evaluations only refresh angles and matrices.
#pragma once

#include <stdint.h>

#include <memory>
#include <vector>

#include "qsv_internal.h"

namespace qsv {

enum GateKind : int32_t {
    K_H = 0, K_HY = 1, K_X = 2, K_CNOT = 3, K_SWAP = 4, K_RZ = 5, K_RY = 6, K_U3 = 7, K_CU3 = 8,
    K_COUNT = 9
};

struct PassPlan {
    TileGeom geom;
    int op_begin = 0, op_end = 0;
    bool global = false;  // fallback: single rotation group applied pairwise over HBM
    uint64_t flip = 0;
    int block_begin = 0, block_end = 0;  // register blocks (m >= 4)
    uint16_t store_cols[12] = {0};       // final SMEM map of the pass (swizzled)
    uint16_t store_t = 0;
    bool map_permuted = false;           // final map differs from the identity
};

struct ParamFill {
    int offset;    // into params
    int src;       // gate index
    int kind;      // gate kind
    int ctrl = 0;  // 1: OP_U1C -- two matrices (control bit 0 / 1), 16 doubles
};

// Controlled-phase deferral of a U3 whose qubit t next acts as a CNOT TARGET
// (the case PhaseDefer cannot take): its phase diag(1, e^{ib}) on t passes the
// CNOT(c, t) as e^{ib (x_t ^ x_c)} = e^{ib x_t} e^{ib x_c} e^{-2ib x_c x_t}:
// the first factor joins the next U3 on t (lambda += b), the second the next
// U3 on c (lambda += b), the third makes that U3 on c controlled by x_t
// (lambda += b - 2b when x_t = 1: OP_U1C), applied before the U3 on t.  The
// source then needs no phase at all (U3Norm shear, 8 FP64 per pair).
struct CzDefer {
    int src;   // deferring U3 (on t)
    int tgt;   // next U3 on t (lambda += b)
    int ctl;   // next U3 on c, becomes OP_U1C controlled by t
};

// Phase deferral of a U3 whose qubit next acts as a CNOT control and then
// receives another U3: U3(t,p,l) = diag(1, e^{ip}) V(t,l) with
// V = [[c, -e^{il} s], [s, e^{il} c]] (two real entries: 12 DFMA per pair
// instead of 14), and diag(1, e^{ip}) commutes with the CNOT control, so it is
// folded into the receiving U3 as l' = l + p.  Decided from structure; the
// angles are applied when parameters are materialised.
struct PhaseDefer {
    int src;   // deferring U3 gate index (applied as V)
    int dst;   // receiving U3 gate index (lambda += phi of src)
};

// A fused same-flip rotation group (OP_GMAT): the table of 2 x 2^(w-1)
// complex 2x2 matrices is rebuilt from the angles on every call.
struct GmatFill {
    int offset;        // params offset of the table
    int r0, r1;        // rotations (in order) of the group
    int F, H, w;       // block-local flip, its highest bit, popcount
    std::vector<uint8_t> yF;  // block-local Y bits of each rotation
};

// A dense-fused gate cluster: a run of gates confined to <= 2 qubits whose
// product is applied as one 2x2 (qb < 0) or 4x4 (rows = 2*bit(qa) + bit(qb))
// matrix, recomputed from the bound values on every call.
struct ClusterFill {
    int offset;               // params offset of the fused matrix
    int qa, qb;               // physical qubits (qb = -1: single-qubit cluster)
    std::vector<int> gates;   // source gate indices, in application order
};

// Small-state rotation program (qsv_small.cu): a state of <= kSmallMaxQubits
// qubits made only of Pauli rotations runs as ONE CTA that keeps the whole
// state in shared memory and walks the same-flip rotation groups (several
// pairs per thread per group), instead of tile passes whose
// straight-line code would stream through one SM's instruction cache.
constexpr int kSmallMaxQubits = 12;
constexpr int kSmallMinQubits = 8;
struct SmallGroup {    // 48 B
    uint32_t xm;       // flip mask (X and Y positions) shared by the group
    // phase masks over the PAIR index p (lo = p with a 0 inserted at bit h):
    // the basis of the rotations' phase-mask differences b0..b2 (0: unused)
    // and the first rotation's phase mask z0, each with bit h removed --
    // parity(lo & m) = parity(p & pm), so a pair's config is linear in p
    uint32_t pm[4];
    // share vectors (amplitude space, bit h = 0, parity(lu & pm[j]) = 0): the
    // pairs lo0 ^ span(lu) share lo0's config, so one thread applies them with
    // one matrix load; chosen inside the group's warp-run subspace
    uint32_t lu[2];
    int32_t h;         // pivot of xm: its highest bit (bit h of lo = 0)
    int32_t r0, r1;    // rotations [r0, r1) in application order
    int32_t dimb;      // number of basis differences (configs = 2^dimb, x 2 for the sign)
};
struct SmallProgram {
    bool valid = false;
    int share = 2;     // log2 pairs per thread sharing a matrix load (1 or 2)
    int ncls = 0;      // invariant GF(2) functionals used: 2^ncls independent classes
    uint32_t w[3] = {0, 0, 0};  // the functionals (amplitude space): parity(i & w_k) is conserved
    std::vector<SmallGroup> groups;
    std::vector<int32_t> meta;    // per rotation: ny mod 4 | (ny odd) << 2 | coordinates << 3
    std::vector<int32_t> src;     // per rotation: its angle is values[3 * src]
    std::vector<int32_t> runs;    // [g0, g1) warp runs (each ends with a CTA barrier)
    // Per-thread addressing, resolved on the host once per structure so the
    // kernel's per-group body is loads, FP64 and stores only:
    //   tab[((g << ncls) | class) * nthr + t] = byte slot of the thread's first
    //     pair's low amplitude | config << 16
    //   xo[4 g .. 4 g + 3] = byte-slot XORs of the other three pairs' lows
    //     (lu0, lu1, lu0 ^ lu1) and of the flip (low -> high amplitude)
    int nthr = 0;
    uint32_t swz[3] = {8u, 8u, 8u};  // shared-memory slot map masks (qsv_small.cu: slot3)
    std::vector<uint32_t> tab;
    std::vector<uint32_t> xo;
    // device copy of the structure-only arrays (groups, meta, runs, xo,
    // tab), uploaded on first use per device; angles go up per evolve
    struct DevCopy {
        int device = -1;
        char *base = nullptr;
        size_t o_groups = 0, o_meta = 0, o_runs = 0, o_xo = 0, o_tab = 0;
        ~DevCopy();
    };
    mutable std::vector<std::shared_ptr<DevCopy>> dev;
};

struct ProgramTemplate {
    int n = 0, m = 0, c = 0;
    SmallProgram small;  // valid: the whole program is rotations on <= 12 qubits
    std::vector<PassPlan> passes;
    std::vector<OpRec> ops;
    std::vector<BlockRec> blocks;
    std::vector<RotRec> rots;      // c/s refreshed per call
    std::vector<int> rot_src;      // theta source index per RotRec
    std::vector<ParamFill> fills;  // matrices refreshed per call
    std::vector<GmatFill> gfills;  // fused group tables refreshed per call
    std::vector<ClusterFill> cfills;  // dense-fused gate clusters refreshed per call
    std::vector<PhaseDefer> defers;   // U3 phase deferrals (see PhaseDefer)
    std::vector<CzDefer> czdefers;    // controlled-phase deferrals (see CzDefer)
    // Normalised U3 forms (see U3Norm in qsv_planner.cpp), per ParamFill:
    // 0 plain, 4 row 0 divided by m00 (m00 = 1), 6 shear (m00 = m11 = 1,
    // both phases deferred); the pass's product of the divisors multiplies
    // its sink fill.
    std::vector<int8_t> fill_mode;
    std::vector<int> fill_pass;
    std::vector<int> pass_sink;       // per pass: ParamFill index of the sink, -1: none
    size_t n_params = 0;
    // global-fallback rotation records (full 64-bit masks), per pass: rots[r0..r1)
    int64_t n_input = 0, n_rotations = 0, n_items = 0, n_fallback = 0, n_blocks = 0;
    int64_t n_fused_gates = 0;  // gates absorbed into dense clusters
    std::vector<int32_t> src_kinds, src_qubits;  // the gate list (cluster materialisation)
};

struct Rot {
    uint64_t x, y, z;
    int src;
};

// Build the small program of a rotation list (false: not eligible).
bool build_small_program(int n, const std::vector<Rot> &R, SmallProgram &sp);

// Build a template from a gate list (kinds/qubits as in qsv_apply_gates).
void plan_gates(int n, int64_t n_gates, const int32_t *kinds, const int32_t *qubits,
                ProgramTemplate &out);
// Build a template from an explicit rotation list.
void plan_rotations(int n, const std::vector<Rot> &rots, int64_t n_input, ProgramTemplate &out);
// Refresh angle-dependent data.  theta_of(src) gives the rotation angle.
void materialize_gates(ProgramTemplate &t, const double *values);
void materialize_rotations(ProgramTemplate &t, const double *theta);
// Fused group tables (after rots[].c/s are refreshed) into params.
void materialize_gmats(const ProgramTemplate &t, double *params);
// Every angle-dependent parameter of a gate-list template (gate matrices,
// fused cluster matrices, fused group tables) into params[t.n_params];
// refreshes t.rots first.
// with_gmats = false: leave the OP_GMAT tables to the device (gmat fill kernel)
// Plain (un-normalised) U3 forms for the next plans of this thread: set when
// a call's angles make a normalised form ill-conditioned (|cos(theta/2)| tiny).
void set_plain_u3(bool on);
bool plain_u3();
// True if the template uses a normalised U3 form these angles cannot take.
bool needs_plain_u3(const ProgramTemplate &t, const double *values);

void materialize_params(ProgramTemplate &t, const double *values, double *params,
                        bool with_gmats = true);
// Gate matrix restatement of circuit.py:198-223 (row-major complex128).
int gate_matrix(int kind, const double *v, double *out);

// ---- expectation sweep plan ----
struct SweepPlan {
    TileGeom geom;
    bool global = false;  // fallback: groups evaluated pairwise over HBM
    std::vector<GroupRec> groups;
    std::vector<TermRec> terms;
    std::vector<int32_t> map;  // sweep-local term -> input term index
    int ndiag = 0;
    std::vector<uint64_t> gflip;  // global fallback: full flip masks per group
};

// jit_layout: Z-only strings get sweeps of their own (the specialised sweep
// kernel handles flip groups only) and flip sweeps hold at most 24 strings.
void plan_expectation(int n, int64_t n_terms, const uint64_t *x, const uint64_t *y,
                      const uint64_t *z, std::vector<SweepPlan> &out, bool jit_layout = false);

// Device-side geometry tables of a tile (see TileDims).
TileDims dims_of(const TileGeom &g);
// comp table: [0..31] tile-index bit positions, [32..43] final map columns,
// [44] final map translation (identity unless a PassPlan is given).
void geom_tables(const TileGeom &g, std::vector<uint64_t> &offhi, std::vector<int32_t> &comp64,
                 const PassPlan *pp = nullptr);

uint64_t hash_structure(int n_qubits, int64_t n_gates, const int32_t *kinds, const int32_t *qubits);

// pauli_evolution blocks recognised in a gate list (the planner's matcher):
// gates [start, start + len) equal exp(-i theta/2 P(x, y, z)), theta = the
// bound value of gate rz.
struct RotSpan {
    int64_t start, len;
    uint64_t x, y, z;
    int64_t rz;
};
void match_rotations(int64_t n_gates, const int32_t *kinds, const int32_t *qubits, std::vector<RotSpan> &out);

}  // namespace qsv
