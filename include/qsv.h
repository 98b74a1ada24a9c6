/*
 * qsv.h -- C ABI of the B200 (sm_100a) state-vector engine (libqsv.so).
 *
 * Drop-in boundary for the state-vector hot path of vqekit
 * (/root/reference/pkg/src/vqekit).  Every entry point names the reference
 * interface it replaces (file:line, relative to /root/reference/pkg/src/vqekit).
 *
 * Conventions
 *  - A state is 2^n complex128 amplitudes; basis-index bit k is qubit k
 *    (statevector.py:1-6).  Host buffers are interleaved (re, im) doubles in
 *    index order -- the little-endian <c16 layout of dump_state
 *    (statevector.py:214-216).  Pin host buffers for full PCIe speed.
 *  - Device memory is owned by the handle; host pointers are borrowed for
 *    the duration of the call only.  All work of all states on one device
 *    is ordered on that device's library stream (qsv_get_stream): states
 *    share the device's scratch, pinned staging buffer and specialised
 *    kernels' __constant__ banks, so one stream per device is what keeps them
 *    race-free.  Calls that return host values synchronise that stream.
 *  - Every call returns QSV_OK (0) or an error code; qsv_last_error() gives a
 *    thread-local message.  The Python layer maps codes to the reference's
 *    exception types (errors.py:9-22; ValueError / ArithmeticError).
 *  - Gate kinds are the reference's closed gate set (circuit.py:27-34):
 *    H=0 HY=1 X=2 CNOT=3 SWAP=4 RZ=5 RY=6 U3=7 CU3=8.  For two-qubit gates the
 *    first qubit is the control / most-significant bit of the 4x4 matrix
 *    (circuit.py:5-6).
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    call fails with QSV_ERR_CUDA.
 */
#ifndef QSV_H
#define QSV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QSV_ABI_VERSION 1

#define QSV_OK 0
#define QSV_ERR_INVALID 1  /* bad argument (ValueError) */
#define QSV_ERR_CUDA 2     /* CUDA runtime failure / no device */
#define QSV_ERR_NOMEM 3    /* device or pinned allocation failed */
#define QSV_ERR_RESOURCE 4 /* request exceeds a hard cap (ResourceLimitError) */

typedef struct qsv_state qsv_state;

/* Plan statistics of the last qsv_apply_gates / qsv_apply_pauli_rotations /
 * qsv_expectation call on the calling thread. */
typedef struct qsv_plan_stats {
    int64_t n_input_ops;   /* gates or rotations or terms passed in */
    int64_t n_rotations;   /* evolution blocks recognised as Pauli rotations */
    int64_t n_items;       /* scheduled items (gates + rotation groups / term groups) */
    int64_t n_passes;      /* HBM passes launched (each reads + writes, or reads, every amplitude) */
    int64_t n_fallback;    /* passes that had to use the global (non-tile) kernel */
    int32_t tile_bits;     /* qubits resident per shared-memory tile */
    int32_t cache_hit;     /* 1 if the structural plan came from the cache */
} qsv_plan_stats;

int qsv_abi_version(void);
const char *qsv_last_error(void);
int qsv_device_count(int *out);
/* Free / total device memory (cudaMemGetInfo): lets callers reject a state
 * that cannot fit before allocating it (statevector.py:47-50 rejects
 * oversized states up front with ResourceLimitError). */
int qsv_mem_info(int device, uint64_t *free_bytes, uint64_t *total_bytes);

/* Handle lifetime.  qsv_create allocates 16 * 2^n bytes on `device` and
 * leaves the amplitudes uninitialised.  (StateVector, statevector.py:26-39) */
int qsv_create(qsv_state **out, int n_qubits, int device);
int qsv_destroy(qsv_state *s);
int qsv_n_qubits(const qsv_state *s, int *out);
/* Cross-process relayout exchange (replaces the NCCL chunk send/recv of the
 * reference-free sharded path, distributed.py; the reference itself has no
 * sharding -- SPEC.md:398).  qsv_ipc_get_handle exports the state's device
 * buffer (QSV_IPC_HANDLE_BYTES bytes); a partner process maps it with
 * qsv_ipc_open and swaps chunks in place with qsv_swap_peer (amplitude
 * offsets, n amplitudes; the peer range is the caller's to keep in bounds and
 * ordered against the peer's own work).  qsv_swap_info: swap kernels run. */
#define QSV_IPC_HANDLE_BYTES 64
int qsv_ipc_get_handle(const qsv_state *s, void *handle);
int qsv_ipc_open(int device, const void *handle, void **peer_base);
int qsv_ipc_close(int device, void *peer_base);
int qsv_swap_peer(qsv_state *s, uint64_t local_offset, void *peer_base, uint64_t peer_offset, uint64_t n);
int qsv_swap_info(int64_t *launches);

/* qsv_set_stream: order this state's later work after everything already
 * queued on cuda_stream (an event fence; NULL = no-op).  Library work still
 * runs on the device's library stream, returned by qsv_get_stream -- wait on
 * it (e.g. torch.cuda.ExternalStream) before consuming qsv_device_ptr data. */
int qsv_set_stream(qsv_state *s, void *cuda_stream);
int qsv_get_stream(const qsv_state *s, void **cuda_stream);
int qsv_device_ptr(const qsv_state *s, void **ptr);   /* zero-copy view (DLPack/torch) */
int qsv_synchronize(qsv_state *s);

/* StateVector.copy (statevector.py:38-39) / the copy in evolve (statevector.py:71). */
int qsv_copy(qsv_state *dst, const qsv_state *src);
/* init_state (statevector.py:42-54): |index>. */
int qsv_set_basis(qsv_state *s, uint64_t index);
/* Host <-> device in dump_state layout (statevector.py:214-216). */
int qsv_upload(qsv_state *s, const double *host);
int qsv_download(const qsv_state *s, double *host);
/* Asynchronous qsv_download: the copy runs on a separate copy stream once the
 * state's queued work is done, overlapping work queued afterwards on other
 * states (pinned host buffers give a truly asynchronous copy).  The state may
 * keep being used: the next call that modifies or frees it first waits for
 * the copy.  qsv_download_wait blocks until the host buffer is complete. */
int qsv_download_async(qsv_state *s, double *host);
int qsv_download_wait(qsv_state *s);

/* kernels.apply_1q (kernels/__init__.py:21; _cykernels.pyx:19-38): m = 2x2 row-major complex128. */
int qsv_apply_1q(qsv_state *s, const double *m, int qubit);
/* kernels.apply_2q (kernels/__init__.py:22; _cykernels.pyx:41-73): m = 4x4, rows 2*bit(q0)+bit(q1). */
int qsv_apply_2q(qsv_state *s, const double *m, int q0, int q1);
/* General dense k-qubit gate, k = 1..5 (north_star (1): up to k local
 * qubits as one 2^k x 2^k block).  m: 2^k x 2^k complex128 row-major; the
 * row / column index is formed from the targets with qubits[0] as the most
 * significant bit -- the apply_2q convention (_cykernels.pyx:41-73,
 * circuit.py:5-6) extended to k qubits.  k = 1, 2 reproduce apply_1q /
 * apply_2q.  Errors: duplicate or out-of-range qubits -> QSV_ERR_INVALID,
 * k > 5 -> QSV_ERR_RESOURCE. */
int qsv_apply_matrix(qsv_state *s, int k, const int32_t *qubits, const double *m);
/* kernels.apply_pauli (kernels/__init__.py:23; _cykernels.pyx:76-102): dst = P src. */
int qsv_apply_pauli(const qsv_state *src, qsv_state *dst, uint64_t x, uint64_t y, uint64_t z);

/* evolve's gate loop (statevector.py:65-74 via _apply_gate :57-62) for a bound
 * circuit: kinds[g], qubits[2g..2g+1] (second = -1 for 1q gates),
 * values[3g..3g+2] (bound parameter values, circuit.py:106-109).  The engine
 * recognises pauli_evolution blocks (circuit.py:271-281) as direct Pauli
 * rotations, fuses everything into shared-memory tile passes and applies it
 * in place.  stats may be NULL. */
int qsv_apply_gates(qsv_state *s, int64_t n_gates, const int32_t *kinds, const int32_t *qubits,
                    const double *values, qsv_plan_stats *stats);

/* Product of exp(-i theta_r / 2 P_r), r = 0..n-1 in order (P_r given by X/Y/Z
 * bit masks as in statevector._string_masks, statevector.py:77-88).  Equals
 * evolve() of pauli_evolution(P_r, -theta_r/2) blocks (circuit.py:254-281). */
int qsv_apply_pauli_rotations(qsv_state *s, int64_t n, const uint64_t *x, const uint64_t *y,
                              const uint64_t *z, const double *theta, qsv_plan_stats *stats);

/* expectation (statevector.py:98-110): out = sum_t c_t <psi|P_t|psi>.
 * out_re receives the real part, out_im the imaginary residue contributed by
 * Im(c_t) (the caller raises above 1e-10, statevector.py:108-109).
 * per_term (nullable, n_terms doubles) receives <psi|P_t|psi> (real). */
int qsv_expectation(const qsv_state *s, int64_t n_terms, const uint64_t *x, const uint64_t *y,
                    const uint64_t *z, const double *coef_re, const double *coef_im,
                    double *out_re, double *out_im, double *per_term, qsv_plan_stats *stats);

/* apply_operator (statevector.py:113-121): dst = sum_t c_t P_t src. */
int qsv_apply_operator(const qsv_state *src, qsv_state *dst, int64_t n_terms, const uint64_t *x,
                       const uint64_t *y, const uint64_t *z, const double *coef_re,
                       const double *coef_im);

/* np.vdot(a, b) (engine.py:74-75, statevector.py:107): out2 = {re, im}. */
int qsv_vdot(const qsv_state *a, const qsv_state *b, double *out2);
/* StateVector.norm (statevector.py:35-36). */
int qsv_norm(const qsv_state *s, double *out);
/* y = alpha*y + beta*x (axpy of apply_operator, statevector.py:120). */
int qsv_axpby(qsv_state *y, const qsv_state *x, double alpha_re, double alpha_im, double beta_re,
              double beta_im);

/* sample (statevector.py:124-147) after the caller's basis rotation: draw
 * `shots` outcomes from |psi|^2 exactly as numpy's
 * Generator(Philox(seed)).choice(2^n, shots, p=|psi|^2/sum) does (cumsum cdf,
 * 53-bit uniforms of the Philox4x64-10 stream with key philox_key[2] =
 * Philox(seed).state['key'], searchsorted 'right'); out_mean = mean of
 * (-1)^{popc(outcome & support_mask)}.  outcomes (nullable, shots int64)
 * receives the drawn basis indices. */
int qsv_sample_parity(const qsv_state *s, uint64_t support_mask, int64_t shots,
                      const uint64_t *philox_key, double *out_mean, int64_t *outcomes);

/* Reverse-mode gradient of a Pauli-rotation product (statevector.py:153-211
 * restricted to circuits made of pauli_evolution blocks, circuit.py:254-281):
 * on entry phi = U|psi0>, lam = H U|psi0> with U = prod_r exp(-i theta_r/2 P_r)
 * (r = 0..R-1 in application order); on return grad[r] = dE/dtheta_r of
 * E = <psi0|U^dag H U|psi0>, phi = |psi0> and lam = U^dag H U|psi0> (both
 * un-rotated in place on the device; the host reads grad once). */
int qsv_rotation_adjoint(qsv_state *phi, qsv_state *lam, int64_t R, const uint64_t *x,
                         const uint64_t *y, const uint64_t *z, const double *theta, double *grad);

/* Prepared programs: qsv_prepare_gates validates and plans a gate structure
 * (kinds / qubits as for qsv_apply_gates) once and returns an id;
 * qsv_apply_prepared(s, id, values) then runs it with new parameter values
 * (3 per gate) without the per-call structure lookup -- the bind-and-evolve
 * loop of vqe_minimize (engine.py:455-457).  Ids stay valid until released. */
int qsv_prepare_gates(int n_qubits, int64_t n_gates, const int32_t *kinds, const int32_t *qubits,
                      int64_t *program_id);
int qsv_apply_prepared(qsv_state *s, int64_t program_id, const double *values,
                       qsv_plan_stats *stats);
int qsv_release_program(int64_t program_id);
/* evolve from a basis state (statevector.py:65-74 with init_state, :42-54):
 * s = gates |index>.  Fused: the first specialised pass synthesises |index>
 * instead of reading the state (saves one full write + read of the vector). */
int qsv_evolve_basis(qsv_state *s, uint64_t index, int64_t n_gates, const int32_t *kinds,
                     const int32_t *qubits, const double *values, qsv_plan_stats *stats);
int qsv_evolve_basis_prepared(qsv_state *s, uint64_t index, int64_t program_id,
                              const double *values, qsv_plan_stats *stats);

/* Planner only (no device work; usable without a GPU): the plan that
 * qsv_apply_gates / qsv_expectation would execute for these inputs. */
int qsv_plan_gates(int n_qubits, int64_t n_gates, const int32_t *kinds, const int32_t *qubits,
                   qsv_plan_stats *out);
int qsv_plan_expectation(int n_qubits, int64_t n_terms, const uint64_t *x, const uint64_t *y,
                         const uint64_t *z, qsv_plan_stats *out);

/* The planner's recognition of pauli_evolution blocks (circuit.py:271-281):
 * count receives the number of blocks; the first min(count, cap) are written
 * as spans[3k..3k+2] = {first gate, gate count, index of the RZ gate whose
 * bound value is theta} and masks[3k..3k+2] = {x, y, z} of P (the block is
 * exp(-i theta/2 P)).  Used by the sharded path to schedule rotations whose
 * flips avoid the global qubits as local work.  No device work. */
int qsv_match_rotations(int n_qubits, int64_t n_gates, const int32_t *kinds, const int32_t *qubits,
                        int64_t cap, int64_t *spans, uint64_t *masks, int64_t *count);

/* ---- multi-device state (one process, P = 2^g shards) --------------------
 * The single-process counterpart of the sharded path (distributed.py; the
 * reference's own parallelism is one process with forked workers,
 * engine.py:169-199): rank r keeps the 2^(n-g) amplitudes whose physical
 * index bits [n-g, n) equal r on device_ids[r] (ids may repeat: several
 * shards on one device).  Gate lists are cut into local segments by the
 * light-cone scheduler with qubit-swap relayouts (pairwise chunk exchange,
 * cudaMemcpyPeerAsync over NVLink / NVSwitch) between them; a logical ->
 * physical qubit map is kept, never swapped back.  qsv_dist_set_basis is lazy
 * (init_state, statevector.py:42-54); qsv_dist_expectation reduces the ranks'
 * partials in ascending order (engine.py:199); qsv_dist_download returns the
 * logical amplitudes in dump_state order (statevector.py:214-216). */
typedef struct qsv_dist qsv_dist;
int qsv_dist_create(qsv_dist **out, int n_qubits, int n_ranks, const int *device_ids);
int qsv_dist_destroy(qsv_dist *d);
int qsv_dist_set_basis(qsv_dist *d, uint64_t index);
int qsv_dist_apply_gates(qsv_dist *d, int64_t n_gates, const int32_t *kinds, const int32_t *qubits,
                         const double *values);
int qsv_dist_expectation(qsv_dist *d, int64_t n_terms, const uint64_t *x, const uint64_t *y,
                         const uint64_t *z, const double *coef_re, const double *coef_im,
                         double *out_re, double *out_im);
int qsv_dist_download(qsv_dist *d, double *host);
/* ranks, local qubits, relayouts so far, bytes each rank sent, qubit map
 * (perm[q] = physical position of logical qubit q; any pointer may be NULL) */
int qsv_dist_info(const qsv_dist *d, int *n_ranks, int *local_qubits, int64_t *relayouts,
                  int64_t *bytes_sent_per_rank, int32_t *perm);
/* whether relayouts swap chunks in place over peer memory (every device pair
 * can address the other, or shards share a device), and how many swap kernels
 * have run; QSV_DIST_P2P=0 forces cudaMemcpyPeerAsync through staging */
int qsv_dist_p2p_info(const qsv_dist *d, int *p2p, int64_t *swap_launches);

/* Debug / test export: the specialised (NVRTC) source of tile pass `k` of the
 * plan for this gate list ("" for global / interpreted passes); host only. */
int qsv_debug_pass_source(int n_qubits, int64_t n_gates, const int32_t *kinds, const int32_t *qubits,
                          int64_t k, char *out, int64_t cap, int64_t *needed, int64_t *n_passes);

/* Debug / test export: the specialised (NVRTC) source of sweep `k` of the
 * expectation plan for these strings ("" when that sweep is interpreted);
 * the planner runs on the host, no device needed. */
int qsv_debug_sweep_source(int n_qubits, int64_t S, const uint64_t *x, const uint64_t *y,
                           const uint64_t *z, int64_t k, char *out, int64_t cap, int64_t *needed,
                           int64_t *n_sweeps);

/* Debug: the compiled tile program for a gate list as JSON (planner output
 * consumed by the CPU emulator in tests/).  needed receives the buffer size. */
int qsv_debug_plan_json(int n_qubits, int64_t n_gates, const int32_t *kinds,
                        const int32_t *qubits, const double *values, char *out, int64_t cap,
                        int64_t *needed);

/* Run-time specialised tile passes (NVRTC-compiled per pass structure):
 * available = 1 if NVRTC + the driver API could be loaded, launches = number
 * of specialised pass launches so far in this process.  Env: QSV_JIT=0
 * disables, QSV_JIT_MIN_QUBITS (default 22) sets the state size from which
 * passes are specialised. */
int qsv_jit_info(int *available, int64_t *launches);

/* Small-state rotation programs: a program made only of Pauli rotations on
 * <= 12 qubits (config 1) runs as one CTA with the state in shared memory
 * instead of tile passes (replaces the same statevector.py:65-74 gate loop).
 * launches = number of such launches so far in this process.  Env:
 * QSV_SMALL=0 runs these programs as tile passes. */
int qsv_small_info(int64_t *launches);

/* Parity-reduced states: an evolve from a basis state by a rotation program
 * whose flips all have even weight (particle-number-conserving ansatze)
 * never leaves the basis state's index-parity class, so the half of the
 * state in that class is evolved as an (n-1)-qubit state (statevector.py's
 * ParityReduced).  dst (n qubits) = the full state: dst[j] = half[j without
 * bit n-1] when parity(j & (wlow | 2^(n-1))) = cls, else 0.  Replaces the
 * full-size gate loop of statevector.py:65-74 for such programs; the reduced
 * result is exactly the reference's. */
int qsv_embed_parity(qsv_state *dst, const qsv_state *half, uint64_t wlow, int cls);

/* Statistics of the last plan on the calling thread (see qsv_plan_stats). */
int qsv_last_plan_stats(qsv_plan_stats *out);

#ifdef __cplusplus
}
#endif

#endif /* QSV_H */
