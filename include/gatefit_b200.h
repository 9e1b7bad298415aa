/*
 * gatefit_b200.h -- C ABI of libgfcuda.so, the B200 (sm_100a) matrix-free
 * contraction engine that is a drop-in for the hot path of the reference
 * `gatefit` package (arXiv 2506.23775).
 *
 * Plain pointers and sizes only.  Device pointers are raw CUDA device
 * addresses (complex128 = two doubles, re then im); `stream` is a cudaStream_t
 * (NULL = legacy default stream).  All calls are asynchronous on `stream`
 * unless stated otherwise.  Every call returns a gf_status; on failure
 * gf_last_error() returns a thread-local message.  Error mapping used by the
 * Python layer mirrors the reference's exceptions:
 *   GF_EINVAL    -> ValueError          (reference kernels.py:75-79, 115-124, 500-501)
 *   GF_ENONFINITE-> FloatingPointError  (reference objective.py:575-578)
 *   GF_ECUDA     -> RuntimeError,  GF_ENOMEM -> MemoryError
 *
 * Conventions (reference kernels.py:1-22): qubit 0 is the most significant
 * bit; a gate on targets (t1, t2) has matrix index 2*bit(t1) + bit(t2);
 * targets with t1 > t2 are normalised internally by the wire swap
 * [0,2,1,3] and outputs are returned in the caller's (t1, t2) orientation.
 */
#ifndef GATEFIT_B200_H
#define GATEFIT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GF_OK = 0,
    GF_EINVAL = 1,
    GF_ENONFINITE = 2,
    GF_ECUDA = 3,
    GF_ENOMEM = 4
} gf_status;

/* Thread-local description of the last failure on this thread. */
const char *gf_last_error(void);
/* ABI version (major*100 + minor). */
int gf_abi_version(void);

/* ------------------------------------------------------------------ *
 * Kernel-level operations.  Each replaces one public op of the
 * reference's kernels.py (file:line given) and is batched over `nvec`
 * contiguous vectors of length 2^k.
 * ------------------------------------------------------------------ */

/* out = G in for every vector (out may equal in: in-place).
 * Replaces kernels.apply_gate (kernels.py:484-515) and the numba cores
 * _apply_{adjacent,general}_{kernel,plain,parity} (kernels.py:132-205,
 * 283-322).  mat: host pointer to 16 complex (32 doubles), row-major.
 * parity_sparse != 0 skips the 8 structurally zero entries. */
int gf_apply_gate(const void *in, void *out, int k, int t1, int t2, const double *mat, int parity_sparse,
                  int64_t nvec, void *stream);

/* out = g in for a one-qubit gate g (host pointer to 4 complex = 8 doubles,
 * row-major 2x2) on qubit q of every vector (out may equal in).  North-star
 * item (1); the reference absorbs one-qubit gates into its two-qubit gates
 * (SPEC.md:102), so the oracle is reference apply_gate with kron(g, I)
 * (kernels.py:484-515).  Same 256-bit streaming paths as gf_apply_gate. */
int gf_apply_gate_1q(const void *in, void *out, int k, int q, const double *mat, int64_t nvec, void *stream);

/* Parity-controlled one-qubit gate of the parity-sector compressed space
 * (no reference counterpart): a 4x4 parity-conserving gate
 * on full-space qubits (a, k_full-1) acting on the compressed vector of
 * k_full-1 bits; `sector` 0 = even, 1 = odd.  mat in the (a, k_full-1)
 * orientation. */
int gf_apply_gate_sector_c1q(const void *in, void *out, int k_full, int a, int sector, const double *mat,
                             int64_t nvec, void *stream);

/* D[4][4] = sum_env bra(i) ket(j) (bra not conjugated) summed over the nvec
 * vector pairs; written to out_dev (16 complex).  Replaces
 * kernels.hole_contract (kernels.py:518-537, core kernels.py:208-242). */
int gf_hole_contract(const void *bra, const void *ket, int k, int t1, int t2, int64_t nvec, void *out_dev,
                     void *stream);

/* out[phys][a] (arity fastest): psi with target bits := j_a, supported where
 * target bits == i_a, a over support (flat 4*i+j, host array).  Replaces
 * kernels.hole_apply (kernels.py:540-565, core kernels.py:245-280). */
int gf_hole_apply(const void *psi, void *out, int k, int t1, int t2, const int64_t *support, int arity,
                  void *stream);

/* Gate applied to each of `arity` interleaved vectors ([2^k][arity]).
 * Replaces kernels.apply_gate_to_array (kernels.py:574-597, cores
 * kernels.py:325-414).  out must not alias in. */
int gf_apply_gate_to_array(const void *in, void *out, int k, int arity, int t1, int t2, const double *mat,
                           int parity_sparse, void *stream);

/* B[a][c] = hole_contract(bra, arr[:, a], targets).flat[support[c]], written
 * to out_dev as [arity][ncols] complex.  Replaces kernels.hole_contract_array
 * (kernels.py:600-623, core kernels.py:417-458). */
int gf_hole_contract_array(const void *bra, const void *arr, int k, int arity, int t1, int t2,
                           const int64_t *support, int ncols, void *out_dev, void *stream);

/* ------------------------------------------------------------------ *
 * Parity-sector index maps and lattice-translation folding (new; SURVEY
 * 8(a) a43/a44).  Bit-exact integer maps over device int64 arrays.
 * ------------------------------------------------------------------ */
/* full index x = (i << 1) | ((popcount(i) & 1) ^ sector) */
int gf_sector_unrank(const int64_t *idx_dev, int64_t m, int sector, int64_t *out_dev, void *stream);
/* i = x >> 1 */
int gf_sector_rank(const int64_t *x_dev, int64_t m, int64_t *out_dev, void *stream);
/* canonical representative (min over 2-site shifts of both spin chains of
 * L sites) and orbit size of full indices x (k = 2L qubits). */
int gf_orbit_canon(const int64_t *x_dev, int64_t m, int L, int64_t *rep_dev, int64_t *size_dev, void *stream);
/* mark[i] = orbit size if compressed index (i0 + i) is the canonical rep of
 * its orbit, else 0; for building the folded basis of the sector. */
int gf_sector_orbit_mark(int64_t i0, int64_t m, int L, int sector, int32_t *mark_dev, void *stream);

/* ------------------------------------------------------------------ *
 * Engine: one plan per circuit topology and device.  Replaces the jitted
 * pass drivers _value_chunk / _gradient_chunk / _hvp_chunk
 * (objective.py:291-337, 432-482) and the chunk protocol of
 * parallel_reduce (objective.py:490-558) for one rank's share of the
 * basis sum.
 * ------------------------------------------------------------------ */
typedef struct gf_plan gf_plan;

enum { GF_VALUE = 1, GF_GRAD = 2, GF_HVP = 4 };

/* t1/t2/logical: per slot, as in the reference Circuit (circuit.py:30-67).
 * sector: -1 = full space (reference semantics), 0/1 = even/odd parity
 * sector compressed on qubit k-1.  max_batch: summands per gf_plan_eval
 * call.  chunk_states: summands per output chunk (the reference uses 64,
 * objective.py:75); every batch must start on a chunk boundary. */
int gf_plan_create(gf_plan **plan, int k, int sector, int n_slots, const int32_t *t1, const int32_t *t2,
                   const int32_t *logical, int n_logical, int64_t max_batch, int chunk_states);
/* Logical gate matrices [n_logical][4][4] complex (host), caller orientation
 * of each logical gate (the reference's logical_gates[i].matrix). */
int gf_plan_set_gates(gf_plan *plan, const double *mats);
/* HVP directions Z per logical gate [n_logical][4][4] complex (host). */
int gf_plan_set_directions(gf_plan *plan, const double *zmats);
/* nd (<= 3) HVP directions [nd][n_logical][4][4] evaluated together: the
 * fused engine shares the psi / bra sweeps across them (full-Hessian columns,
 * reference objective.py:701-767).  gf_plan_eval records then carry nd H
 * blocks: rec = 2 + 32*n_logical*(1 + nd). */
int gf_plan_set_directions_multi(gf_plan *plan, int nd, const double *zmats);
/* Evaluate `nvec` summands.  basis_dev: int64 [nvec] basis indices (in the
 * compressed space when sector >= 0).  weights_dev: double [nvec] or NULL
 * (translation-fold orbit sizes).  phi0_dev: complex [nvec][2^K] target
 * columns conj(U|j>) (K = k, or k-1 with a sector).  out_dev: double
 * [ceil(nvec/chunk_states)][rec] with rec = 2 + 32*n_logical*(1 + nd) doubles:
 *   value (complex), D[n_logical][4][4] (holomorphic, logical orientation,
 *   accumulated over shared slots), H_d[n_logical][4][4] (holomorphic HVP per
 *   direction; nd = 1 unless gf_plan_set_directions_multi);
 * each record is the deterministic sum over its chunk (the reference's
 * _Partial, objective.py:536-558).  value is phi0 . C|j> summed (the
 * objective is f = -Re of the total, objective.py:606). */
int gf_plan_eval(gf_plan *plan, int flags, int64_t nvec, const int64_t *basis_dev, const double *weights_dev,
                 const void *phi0_dev, double *out_dev, void *stream);
/* Per-slot (normalised orientation) derivative sums of the last eval,
 * [n_slots][16] complex each for D and H (device), for tests.  D is only
 * defined when the eval requested GF_GRAD (an HVP-only eval skips the
 * gradient holes, as the reference's _hvp_chunk does), H only with GF_HVP. */
int gf_plan_slot_outputs(gf_plan *plan, int64_t nvec, double *d_dev, double *h_dev, void *stream);
/* Number of this library's kernels launched by the last gf_plan_eval. */
int64_t gf_plan_last_launches(const gf_plan *plan);
/* Phase timing with CUDA events on the eval stream (off by default).
 * Turning it on resets the accumulators; gf_plan_phase_times waits for the
 * last eval and returns accumulated milliseconds and kernel launches of
 * [forward sweep, reverse sweep, ascending sweep, reductions]. */
int gf_plan_set_profiling(gf_plan *plan, int on);
int gf_plan_phase_times(gf_plan *plan, double *ms4, int64_t *launches4);
/* Profiling detail (new): the first reverse pass of the profiled evaluations
 * -- the sweep's dominant launch, every tile live -- accumulated device time
 * in ms, launches, summand vectors processed and the slots of the pass. */
int gf_plan_first_reverse_pass(gf_plan *plan, double *ms, int64_t *launches, int64_t *vectors, int *slots);
/* Engine shape of a plan: fused tile engine on/off, local (tile) bits, number
 * of fused passes per forward / reverse sweep, CTAs per summand. */
int gf_plan_describe(const gf_plan *plan, int *fused, int *tile_bits, int *n_fwd_passes, int *n_rev_passes,
                     int *ctas);

/* Light cone of the basis states (new; no reference counterpart: the
 * reference applies every slot to the whole vector, objective.py:310-337).
 * psi_l = G_l ... G_1 |j> vanishes wherever a qubit no applied slot has touched
 * differs from j, so the fused engine skips the tiles that disagree with j on
 * such a qubit.  frac3 = fraction of the slot work still executed in the
 * forward, reverse and ascending sweeps (1.0 = nothing skipped; GF_LIGHTCONE=0
 * disables the rule). */
int gf_plan_live_fraction(const gf_plan *plan, double *frac3);

/* Host-only query of the fused pass plan (no device work): the passes the
 * engine would run for slots (t1[s], t2[s]) on k qubits (sector -1/0/1) with
 * 2^tile_bits-amplitude tiles; sweep 0 = forward, 1 = reverse.  Writes the
 * pass count, the slots per pass, the slots in execution order and each
 * pass's local bit set.  New (the reference runs one slot at a time,
 * objective.py:255-280); used by the planner tests. */
int gf_plan_layout(int k, int sector, int n_slots, const int32_t *t1, const int32_t *t2, int tile_bits, int sweep,
                   int max_passes, int *n_passes, int *pass_sizes, int *slot_order, unsigned long long *pass_bits);
int gf_plan_destroy(gf_plan *plan);

/* ------------------------------------------------------------------ *
 * Hessian chunk driver: the reference's _hessian_chunk (objective.py:340-423)
 * with its pair CSR (_pair_csr, objective.py:209-247), as consumed by
 * full_hessian's chunk closure (objective.py:729-744).  Full space only (the
 * reference's semantics); cached passes [n+1] x batch x 2^k per direction.
 * ------------------------------------------------------------------ */
typedef struct gf_hess_plan gf_hess_plan;

/* Slots as gf_plan_create.  support[arity]: flat entries 4*i+j of the hole
 * support in logical orientation (16 = DENSE_SUPPORT, 8 = PARITY_SUPPORT,
 * kernels.py:52-58); swapped slots use the remapped support
 * (kernels.py:568-571) internally.  The pair CSR is exactly the reference's
 * _pair_csr output: first_list[nfirst] ascending, first_start[nfirst + 1],
 * and per pair (first_start[nfirst] of them) pair_second (ascending within a
 * first slot), pair_mult (translation-class size with dedup, else 1),
 * pair_route (upper-triangular logical-pair index a*nlog - a(a-1)/2 + (b-a)),
 * pair_sym (same logical gate), pair_flip (first slot's logical gate is the
 * later one).  All host arrays, copied at creation. */
int gf_hess_plan_create(gf_hess_plan **plan, int k, int n_slots, const int32_t *t1, const int32_t *t2,
                        const int32_t *logical, int n_logical, const int64_t *support, int arity,
                        const int64_t *first_list, int64_t nfirst, const int64_t *first_start,
                        const int64_t *pair_second, const double *pair_mult, const int64_t *pair_route,
                        const int32_t *pair_sym, const int32_t *pair_flip, int64_t max_batch, int chunk_states);
/* Logical gates as gf_plan_set_gates; parity_mode != 0 applies parity-sparse
 * slot matrices without their structural zeros (the reference _Plan's sparse
 * flags, objective.py:188). */
int gf_hess_plan_set_gates(gf_hess_plan *plan, const double *mats, int parity_mode);
/* `nvec` summands (basis_dev int64 [nvec], weights_dev double [nvec] or NULL,
 * phi0_dev complex [nvec][2^k]).  out_dev: double [ceil(nvec/chunk)][rec],
 * rec = 2 + 32*n_logical + 2*R*arity*arity, R = n_logical(n_logical+1)/2:
 *   value (complex), D[n_logical][4][4] (holomorphic, logical orientation),
 *   block_acc[R][arity][arity] (complex, the reference's routed layout);
 * each record the deterministic sum over its chunk.  out_counts: host
 * int64[5] incremented with the reference's counters (objective.py:65-73):
 * gate, array-gate, hole-apply, hole-contract and pair applications. */
int gf_hess_plan_eval(gf_hess_plan *plan, int64_t nvec, const int64_t *basis_dev, const double *weights_dev,
                      const void *phi0_dev, double *out_dev, int64_t *out_counts, void *stream);
/* Per-slot gradient holes of the last eval summed over its nvec summands,
 * [n_slots][4][4] complex in normalised wire orientation (device): the
 * reference's per-chunk dacc (objective.py:329-336). */
int gf_hess_plan_slot_outputs(gf_hess_plan *plan, int64_t nvec, double *d_dev, void *stream);
int64_t gf_hess_plan_last_launches(const gf_hess_plan *plan);
int gf_hess_plan_destroy(gf_hess_plan *plan);

/* ------------------------------------------------------------------ *
 * Matrix-free target oracle (replaces the CPU
 * KrylovOracle / DenseOracle of reference models.py:305-393 as the
 * producer of phi0 = conj(exp(-iHt)|j>)).  Terms are two-site operators
 * (ta[t], tb[t]) with coefficient coef[t]: hop[t] != 0 is
 * |01><10| + |10><01| (models.py:40-42), else n_a n_b (models.py:44).
 * ------------------------------------------------------------------ */
/* out = H in for nvec full-space vectors (out must not alias in). */
int gf_hamiltonian_apply(const void *in, void *out, int k, const int32_t *ta, const int32_t *tb, const double *coef,
                         const int32_t *hop, int nterms, int64_t nvec, void *stream);
/* One Chebyshev order with H~ = scale*H + shift on nvec stored vectors:
 * t_next = H~ t_cur (t_prev NULL) or 2 H~ t_cur - t_prev, then
 * acc += c t_next (acc nullable).  sector_flags bits 0-1: 3 = full space,
 * 0/1 = even/odd compressed sector; bit 8: accumulate conj(c t_next). */
int gf_cheb_step(const void *t_cur, const void *t_prev, void *t_next, void *acc, int k, const int32_t *ta,
                 const int32_t *tb, const double *coef, const int32_t *hop, int nterms, double scale, double shift,
                 double c_re, double c_im, int64_t nvec, int sector_flags, void *stream);

/* Number-block target oracle: exp(-iHt)|j> inside j's particle-number block
 * (hopping conserves the occupation of each connected component of the hop
 * graph).  desc = [k, ncomp, then per component: L, n, qubit_0..qubit_{L-1}];
 * block vectors are indexed by the mixed-radix colex ranks of the component
 * patterns.  terms = [kind (0 hop, 1 nn), comp_a, local_a, comp_b, local_b]
 * per term, coef per term.  gf_nb_cheb_step: one Chebyshev order as in
 * gf_cheb_step; gf_nb_scatter: block vectors cols[colidx[b]] -> zeroed rows
 * rows[rowidx[b]], dense (sector -1) or sector-compressed (null maps mean the
 * identity); gf_nb_rank: block indices of full-space states of the block. */
int gf_nb_cheb_step(const void *t_cur, const void *t_prev, void *t_next, void *acc, const int32_t *desc, int ndesc,
                    const int32_t *terms, const double *coef, int nterms, double scale, double shift, double c_re,
                    double c_im, int64_t nvec, void *stream);
int gf_nb_scatter(const void *cols, const int64_t *colidx, void *rows, const int64_t *rowidx, int64_t nrows,
                  int64_t row_len, const int32_t *desc, int ndesc, int sector, void *stream);
int gf_nb_rank(const int64_t *js, int64_t *out, int64_t n, const int32_t *desc, int ndesc, void *stream);
/* Whole block matrix in one launch (row b = sum_m coefs[m] T_m(H~) e_b, block
 * coordinates; one CTA per row, series on chip); D <= 6400; coefs: device
 * array of norder + 1 complex values; work: device scratch of at least
 * D * (16 + 12 * n_hop_terms) bytes. */
int gf_nb_block_matrix(void *out, const int32_t *desc, int ndesc, const int32_t *terms, const double *coef, int nterms,
                       const void *coefs, int norder, double scale, double shift, void *work, void *stream);
/* Rows from precomputed block matrices (all device arrays, no host sync):
 * row b = block row rank_of[j] of block block_of[j] (j = js[b]) scattered to
 * full_of[stoff[blk] + x] >> shift; rows must be zeroed; nrows <= 65535. */
int gf_nb_gather(const int64_t *js, int64_t nrows, const void *mats, const int64_t *matoff, const int64_t *stoff,
                 const int32_t *blkdim, const int32_t *block_of, const int32_t *rank_of, const int64_t *full_of,
                 int64_t max_dim, int shift, void *out, int64_t row_len, void *stream);

/* Synchronous check of n device doubles (engine records): GF_ENONFINITE if
 * any is NaN or Inf, else GF_OK.  The reference raises FloatingPointError on
 * non-finite results (objective.py:575-578, optimizer.py:147-149). */
int gf_check_finite(const double *x_dev, int64_t n, void *stream);

/* Device-memory helpers for bindings without a tensor library (the ctypes
 * stub of INTEGRATION.md).  gf_memcpy kind: 0 = H2D, 1 = D2H, 2 = D2D
 * (asynchronous on `stream`; pair with gf_stream_sync). */
int gf_set_device(int device);
int gf_malloc(void **ptr, int64_t bytes);
int gf_free(void *ptr);
int gf_memcpy(void *dst, const void *src, int64_t bytes, int kind, void *stream);
int gf_stream_sync(void *stream);

/* Measurement helper (bench.py roofline): back-to-back FP64 work on all SMs.
 * which = 0: DMMA m8n8k4 (FP64 tensor cores), 1: DFMA, 2: both interleaved.  *flops receives the
 * flop count of the launch; time it with events on `stream`. */
int gf_peak_fp64(int which, int blocks, int iters, double *sink_dev, double *flops, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GATEFIT_B200_H */
