// gf_hessian.cu -- the reference's Hessian chunk driver on the GPU.
//
// Reference: _hessian_chunk (objective.py:340-423) with the pair CSR of
// _pair_csr (objective.py:209-247), consumed by full_hessian's chunk closure
// (objective.py:729-744).  Per summand j (a batch of summands per launch,
// grid.y = summand):
//   cached passes   psis[l+1] = G_l psis[l], phis[m] = G_{n-m}^T phis[m-1]
//                   (objective.py:307-319)
//   gradient        D_l = hole(phis[n-l-1], psis[l])  (objective.py:329-336)
//   pairs           for every first slot l of the CSR: harr = hole_apply(psis[l])
//                   (kernels.py:245-280), then for l' = l+1 .. last(l):
//                   out_t = hole_contract_array(phis[n-l'-1], cur) at the listed
//                   pairs (kernels.py:417-458), routed into block_acc[route] with
//                   multiplicity and the sym / flip transposes
//                   (objective.py:398-416); cur <- G_l' cur (kernels.py:325-414)
// With translation dedup (circuit.py:173-211) only one representative pair per
// class is contracted and scaled by the class size, and a first slot's array
// is propagated only up to its last listed pair: the work reduction of
// PAPER.md:746.
//
// B200 layout: the caches are [n+1][nvec][N] (one contiguous batch per level),
// hole arrays [nvec][N][A] (arity fastest, as the reference's, so one
// tuple's A values form a 256 B run for A = 16).  The contraction of slot l'
// is fused into the array update of the same slot: one pass reads cur, adds
// its contraction partial and writes G_l' cur.  Partials are per CTA, summed
// in CTA order, then per chunk in summand and pair order -- deterministic
// for any batch size and GPU count.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "gf_common.cuh"
#include "gf_internal.h"

using namespace gf;

namespace {

constexpr int HT = 256;        // threads per CTA
constexpr int HMAXCTAS = 148;  // CTAs per summand for the array passes

struct HSupport {
    int row[16], col[16];  // per support position: target-bit row / column (slot orientation)
};

struct HSlot {
    int lo, hi;       // bit positions, hi > lo
    bool swapped, sparse;
    int logical;
};

#define GF_CUDA(call)                                                                                   \
    do {                                                                                                \
        cudaError_t _e = (call);                                                                        \
        if (_e != cudaSuccess)                                                                          \
            return gf_fail(_e == cudaErrorMemoryAllocation ? GF_ENOMEM : GF_ECUDA, "%s:%d %s (%s)",     \
                           __FILE__, __LINE__, cudaGetErrorName(_e), cudaGetErrorString(_e));           \
    } while (0)

// ---------------------------------------------------------------------------
// cached passes
// ---------------------------------------------------------------------------

// psi_0 = |j>, phis_0 = w phi0
__global__ void kh_init(double2 *psi0, double2 *phi0c, const double2 *phi0, const int64_t *basis,
                        const double *weights, u64 N, int64_t nvec)
{
    const u64 total = N * (u64)nvec;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (u64)gridDim.x * blockDim.x) {
        const u64 b = i / N, x = i - b * N;
        psi0[i] = make_double2((int64_t)x == basis[b] ? 1.0 : 0.0, 0.0);
        const double w = weights ? weights[b] : 1.0;
        phi0c[i] = cscale(phi0[i], w);
    }
}

// out = M in over nvec contiguous vectors of N amplitudes, tuple per thread
template <bool SPARSE>
__global__ void __launch_bounds__(HT) kh_apply(const double2 *__restrict__ in, double2 *__restrict__ out, int logN,
                                               u64 total, int lo, int hi, const Mat4 g)
{
    const int logU = logN - 2;
    const u64 umask = (1ull << logU) - 1ull;
    const u64 ol = 1ull << lo, oh = 1ull << hi;
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (u64)gridDim.x * blockDim.x) {
        const u64 v = t >> logU, r = t & umask;
        const u64 b = (v << logN) | ins0(ins0(r, lo), hi);
        double2 x[4] = {in[b], in[b + ol], in[b + oh], in[b + ol + oh]}, y[4];
        mv4<SPARSE>(g, x, y);
        out[b] = y[0];
        out[b + ol] = y[1];
        out[b + oh] = y[2];
        out[b + ol + oh] = y[3];
    }
}

// gradient hole of one slot for every summand: part[b][cta][32]; the value
// <phi0|psi_n> rides on the last slot's launch (vpart[b][cta][2])
__global__ void __launch_bounds__(HT) kh_hole(const double2 *__restrict__ bra, const double2 *__restrict__ ket,
                                              int logN, int lo, int hi, double *part,
                                              const double2 *__restrict__ vbra, const double2 *__restrict__ vket,
                                              double *vpart)
{
    const u64 N = 1ull << logN, units = N >> 2;
    const u64 vb = (u64)blockIdx.y * N;
    const u64 ol = 1ull << lo, oh = 1ull << hi;
    double acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = 0.0;
    double vre = 0.0, vim = 0.0;
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < units; t += (u64)gridDim.x * blockDim.x) {
        const u64 b = vb + ins0(ins0(t, lo), hi);
        const u64 r[4] = {b, b + ol, b + oh, b + ol + oh};
        double2 x[4], y[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            x[i] = bra[r[i]];
            y[i] = ket[r[i]];
        }
        hole_acc(acc, x, y);
        if (vpart) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const double2 f = vbra[r[i]], s = vket[r[i]];
                vre = fma(f.x, s.x, fma(-f.y, s.y, vre));
                vim = fma(f.x, s.y, fma(f.y, s.x, vim));
            }
        }
    }
    __shared__ double red[HT / 32 * 32];
    const u64 slot = (u64)blockIdx.y * gridDim.x + blockIdx.x;
    const double s = block_reduce32(acc, red);
    if (threadIdx.x < 32) part[slot * 32 + threadIdx.x] = s;
    if (vpart) {
        double a2[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) a2[i] = 0.0;
        a2[0] = vre;
        a2[1] = vim;
        const double v = block_reduce32(a2, red);
        if (threadIdx.x < 2) vpart[slot * 2 + threadIdx.x] = v;
    }
}

// q[b][e] = sum over CTAs ascending of part[b][c][e]
__global__ void kh_reduce(const double *part, double *q, int64_t nb, int ctas, int ne)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nb * ne) return;
    const int64_t b = i / ne;
    const int e = (int)(i - b * ne);
    double acc = 0.0;
    for (int c = 0; c < ctas; ++c) acc += part[(b * ctas + c) * ne + e];
    q[i] = acc;
}

// ---------------------------------------------------------------------------
// hole arrays
// ---------------------------------------------------------------------------

// harr[b][phys][a] = psi_b[phys with target bits := col_a] where target bits
// of phys == row_a, else 0 (kernels.py:245-280).  Thread = (tuple, a).
template <int A>
__global__ void __launch_bounds__(HT) kh_hole_apply(const double2 *__restrict__ psi, double2 *__restrict__ arr,
                                                    int logN, int lo, int hi, const HSupport sup)
{
    const u64 N = 1ull << logN, units = N >> 2;
    const int a = threadIdx.x % A;
    const int ra = sup.row[a], ca = sup.col[a];
    const u64 ol = 1ull << lo, oh = 1ull << hi;
    const u64 vb = (u64)blockIdx.y * N;
    for (u64 t = ((u64)blockIdx.x * blockDim.x + threadIdx.x) / A; t < units;
         t += (u64)gridDim.x * blockDim.x / A) {
        const u64 b = ins0(ins0(t, lo), hi);
        const u64 r[4] = {b, b + ol, b + oh, b + ol + oh};
        const double2 src = psi[vb + r[ca]];
#pragma unroll
        for (int q = 0; q < 4; ++q) arr[(vb + r[q]) * A + a] = (q == ra) ? src : czero();
    }
}

// Fused pair contraction + array update of slot l' for every summand:
// part[b][cta][c][a] = sum over the CTA's tuples of bra(row_c) cur(col_c, a)
// (kernels.py:417-458, stored [c][a] = out_t), and out = G cur when APPLY.
// Thread = (tuple, row i, arity index a): it loads the tuple's four values of
// its a (coalesced over a; the four i-threads of an a share the addresses),
// accumulates bra_i cur_j for j = 0..3 and writes output row i of G cur.  Four
// accumulators per thread instead of A_s keep the kernel register-light; the
// CTA's tuple lanes are summed in shared memory in a fixed order.
template <int A, int AS, bool CONTRACT, bool APPLY, bool SPARSE>
__global__ void __launch_bounds__(HT) kh_pair(const double2 *__restrict__ bra, const double2 *__restrict__ cur,
                                              double2 *__restrict__ out, int logN, int lo, int hi,
                                              const HSupport sup, const Mat4 g, double2 *part)
{
    constexpr int TL = HT / (4 * A);  // tuples per CTA iteration (4 for A = 16, 8 for A = 8)
    const u64 N = 1ull << logN, units = N >> 2;
    const int a = threadIdx.x % A, i = (threadIdx.x / A) & 3, tl = threadIdx.x / (4 * A);
    const u64 ol = 1ull << lo, oh = 1ull << hi;
    const u64 oi = ((i & 1) ? ol : 0ull) + ((i & 2) ? oh : 0ull);
    const u64 vb = (u64)blockIdx.y * N;
    double2 gi[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) gi[j] = g.m[4 * i + j];
    double2 acc[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j] = czero();
    // two tuples per trip, all loads first (memory-level parallelism)
    const u64 stride = (u64)gridDim.x * TL;
    for (u64 t0 = (u64)blockIdx.x * TL + tl; t0 < units; t0 += 2 * stride) {
        double2 x[2][4], y[2];
        u64 bb[2];
        bool ok[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const u64 t = t0 + u * stride;
            ok[u] = t < units;
            const u64 b = vb + ins0(ins0(ok[u] ? t : t0, lo), hi);
            bb[u] = b;
            if (ok[u]) {
                x[u][0] = cur[b * A + a];
                x[u][1] = cur[(b + ol) * A + a];
                x[u][2] = cur[(b + oh) * A + a];
                x[u][3] = cur[(b + ol + oh) * A + a];
                if (CONTRACT) y[u] = bra[b + oi];
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (!ok[u]) continue;
            if (CONTRACT) {
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[j] = cfma(y[u], x[u][j], acc[j]);
            }
            if (APPLY) {
                double2 v;
                if (SPARSE) {  // parity-conserving rows: {0,3} x {0,3} and {1,2} x {1,2}
                    const int j0 = (i == 0 || i == 3) ? 0 : 1, j1 = 3 - j0;
                    v = cfma(gi[j1], x[u][j1], cmul(gi[j0], x[u][j0]));
                } else {
                    v = cmul(gi[0], x[u][0]);
#pragma unroll
                    for (int j = 1; j < 4; ++j) v = cfma(gi[j], x[u][j], v);
                }
                out[(bb[u] + oi) * A + a] = v;
            }
        }
    }
    if (CONTRACT) {
        __shared__ double2 red[TL][4][4][A];  // [tuple lane][j][i][a]
#pragma unroll
        for (int j = 0; j < 4; ++j) red[tl][j][i][a] = acc[j];
        __syncthreads();
        const u64 slot = (u64)blockIdx.y * gridDim.x + blockIdx.x;
        for (int e = threadIdx.x; e < AS * A; e += HT) {
            const int c = e / A, aa = e - c * A;
            double2 s = czero();
#pragma unroll
            for (int q = 0; q < TL; ++q) s = cadd(s, red[q][sup.col[c]][sup.row[c]][aa]);
            part[slot * (AS * A) + e] = s;
        }
    }
}

// Array update without a contraction (kernels.py:325-414): thread = (tuple,
// arity index a) loads the tuple's four values of its a once and writes all
// four outputs (the (tuple, row, a) layout of kh_pair would load them 4x).
template <int A, bool SPARSE>
__global__ void __launch_bounds__(HT) kh_array_apply(const double2 *__restrict__ cur, double2 *__restrict__ out,
                                                     int logN, int lo, int hi, const Mat4 g)
{
    constexpr int TL = HT / A;
    const u64 N = 1ull << logN, units = N >> 2;
    const int a = threadIdx.x % A, tl = threadIdx.x / A;
    const u64 ol = 1ull << lo, oh = 1ull << hi;
    const u64 vb = (u64)blockIdx.y * N;
    const u64 stride = (u64)gridDim.x * TL;
    for (u64 t0 = (u64)blockIdx.x * TL + tl; t0 < units; t0 += 2 * stride) {
        double2 x[2][4];
        u64 r[2][4];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const u64 t = t0 + u * stride;
            if (t >= units) continue;
            const u64 b = vb + ins0(ins0(t, lo), hi);
            r[u][0] = b * A + a;
            r[u][1] = (b + ol) * A + a;
            r[u][2] = (b + oh) * A + a;
            r[u][3] = (b + ol + oh) * A + a;
#pragma unroll
            for (int q = 0; q < 4; ++q) x[u][q] = cur[r[u][q]];
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (t0 + u * stride >= units) continue;
            double2 y[4];
            mv4<SPARSE>(g, x[u], y);
#pragma unroll
            for (int q = 0; q < 4; ++q) out[r[u][q]] = y[q];
        }
    }
}

// per-summand pair result q[b][c][a] (= out_t[c][a]) summed over CTAs
__global__ void kh_pair_reduce(const double2 *part, double2 *q, int64_t nvec, int ctas, int ne)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nvec * ne) return;
    const int64_t b = i / ne;
    const int e = (int)(i - b * ne);
    double2 acc = czero();
    for (int c = 0; c < ctas; ++c) acc = cadd(acc, part[(b * ctas + c) * ne + e]);
    q[i] = acc;
}

// Chunk records rec = [value (2)] [D: nlog*32] [blocks: R*A*A*2]; one warp per
// entry, lanes over the chunk's summands, fixed xor tree.  Blocks follow the
// reference's routing (objective.py:398-416): sym adds out_t^T and out_t,
// flip adds out_t, plain adds out_t^T (block[a][b] = m * out_t[b][a]).
__global__ void kh_records(const double *qD, const double *qV, const double2 *qP, int64_t nvec, int nslots, int nlog,
                           const int *lstart, const int *lslots, const int *swapped, const int *rstart,
                           const int *rpairs, const double *mult, const int *sym, const int *flip, int A, int R,
                           int chunk, double *out)
{
    const int rec = 2 + 32 * nlog + 2 * R * A * A;
    const int64_t nchunks = (nvec + chunk - 1) / chunk;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nchunks * rec) return;
    const int64_t ch = w / rec;
    const int r = (int)(w - ch * rec);
    const int64_t b0 = ch * chunk, b1 = (nvec < b0 + chunk) ? nvec : (b0 + chunk);
    double acc = 0.0;
    if (r < 2) {
        for (int64_t b = b0 + lane; b < b1; b += 32) acc += qV[b * 2 + r];
    } else if (r < 2 + 32 * nlog) {
        const int rr = r - 2, l = rr >> 5, q = rr & 31, e = q >> 1, ri = q & 1, ii = e >> 2, jj = e & 3;
        for (int64_t b = b0 + lane; b < b1; b += 32)
            for (int t = lstart[l]; t < lstart[l + 1]; ++t) {
                const int s = lslots[t];
                int si = ii, sj = jj;
                if (swapped[s]) {  // WIRE_SWAP = [0,2,1,3]
                    si = (ii == 1) ? 2 : (ii == 2 ? 1 : ii);
                    sj = (jj == 1) ? 2 : (jj == 2 ? 1 : jj);
                }
                acc += qD[((int64_t)s * nvec + b) * 32 + 2 * (4 * si + sj) + ri];
            }
    } else {
        const int rr = r - 2 - 32 * nlog;
        const int ri = rr & 1, e = rr >> 1;
        const int route = e / (A * A), ab = e - route * A * A, a = ab / A, bb = ab - a * A;
        for (int64_t b = b0 + lane; b < b1; b += 32)
            for (int t = rstart[route]; t < rstart[route + 1]; ++t) {
                const int p = rpairs[t];
                const double2 *o = qP + ((int64_t)p * nvec + b) * A * A;  // out_t[c][a] at c * A + a
                const double m = mult[p];
                double v;
                if (sym[p]) {
                    const double2 x = o[bb * A + a], y = o[a * A + bb];
                    v = m * (ri ? x.y : x.x) + m * (ri ? y.y : y.x);
                } else if (flip[p]) {
                    const double2 x = o[a * A + bb];
                    v = m * (ri ? x.y : x.x);
                } else {
                    const double2 x = o[bb * A + a];
                    v = m * (ri ? x.y : x.x);
                }
                acc += v;
            }
    }
    acc = warp_sum(acc);
    if (lane == 0) out[w] = acc;
}

// out[a][c] = sum over CTAs of part[cta][c][a] (the public B[a, c] layout of
// kernels.hole_contract_array, kernels.py:600-623)
__global__ void kh_pair_reduce_T(const double2 *part, double2 *out, int ctas, int ncols, int A)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ncols * A) return;
    const int c = i / A, a = i - c * A;
    double2 acc = czero();
    for (int t = 0; t < ctas; ++t) acc = cadd(acc, part[(size_t)t * ncols * A + i]);
    out[a * ncols + c] = acc;
}

// per-slot gradient holes summed over the batch: out[s][32] (normalised
// wire orientation, the reference's dacc)
__global__ void kh_slot_sums(const double *qD, int64_t nvec, int nslots, double *out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nslots * 32) return;
    const int s = i >> 5, e = i & 31;
    double acc = 0.0;
    for (int64_t b = 0; b < nvec; ++b) acc += qD[((int64_t)s * nvec + b) * 32 + e];
    out[i] = acc;
}

}  // namespace

static int grid_units(u64 units, int threads_per_unit)
{
    const u64 ctas = (units * threads_per_unit + HT - 1) / HT;
    return (int)std::max<u64>(1, std::min<u64>(ctas, HMAXCTAS));
}

// ---------------------------------------------------------------------------
// fast paths of the public kernel ops (gf_ops.cu) for arity / support sizes
// 8 and 16: thread = (tuple, arity index), no 64-bit divisions, CTA partials
// summed in CTA order
// ---------------------------------------------------------------------------
static HSupport hsupport(const int *row, const int *col, int n)
{
    HSupport s;
    for (int c = 0; c < 16; ++c) {
        s.row[c] = c < n ? row[c] : 0;
        s.col[c] = c < n ? col[c] : 0;
    }
    return s;
}

int gf_fast_hole_apply(const void *psi, void *out, int k, int lo, int hi, const int *row, const int *col, int arity,
                       void *stream)
{
    const u64 units = (1ull << k) >> 2;
    const dim3 grid(grid_units(units, arity) * 8, 1);
    const HSupport sp = hsupport(row, col, arity);
    cudaStream_t st = (cudaStream_t)stream;
    if (arity == 16) kh_hole_apply<16><<<grid, HT, 0, st>>>((const double2 *)psi, (double2 *)out, k, lo, hi, sp);
    else if (arity == 8) kh_hole_apply<8><<<grid, HT, 0, st>>>((const double2 *)psi, (double2 *)out, k, lo, hi, sp);
    else return gf_fail(GF_EINVAL, "fast hole apply needs arity 8 or 16");
    GF_CUDA(cudaGetLastError());
    return GF_OK;
}

int gf_fast_array_apply(const void *in, void *out, int k, int arity, int lo, int hi, const Mat4 &g, int sparse,
                        void *stream)
{
    const u64 units = (1ull << k) >> 2;
    const dim3 grid(grid_units(units, arity) * 8, 1);
    cudaStream_t st = (cudaStream_t)stream;
    const double2 *x = (const double2 *)in;
    double2 *y = (double2 *)out;
#define KH_ARR(A_, S_) kh_array_apply<A_, S_><<<grid, HT, 0, st>>>(x, y, k, lo, hi, g)
    if (arity == 16) { if (sparse) KH_ARR(16, true); else KH_ARR(16, false); }
    else if (arity == 8) { if (sparse) KH_ARR(8, true); else KH_ARR(8, false); }
    else return gf_fail(GF_EINVAL, "fast array apply needs arity 8 or 16");
#undef KH_ARR
    GF_CUDA(cudaGetLastError());
    return GF_OK;
}

int gf_fast_hole_array(const void *bra, const void *arr, int k, int arity, int lo, int hi, const int *row,
                       const int *col, int ncols, void *out, void *stream)
{
    const u64 units = (1ull << k) >> 2;
    const int ctas = grid_units(units, arity) * 8;
    const dim3 grid(ctas, 1);
    const HSupport sp = hsupport(row, col, ncols);
    cudaStream_t st = (cudaStream_t)stream;
    double2 *part = nullptr;
    GF_CUDA(cudaMallocAsync((void **)&part, sizeof(double2) * (size_t)ctas * ncols * arity, st));
    Mat4 g0;
    memset(&g0, 0, sizeof g0);
    const double2 *b = (const double2 *)bra, *x = (const double2 *)arr;
#define KH_HA(A_, S_) kh_pair<A_, S_, true, false, false><<<grid, HT, 0, st>>>(b, x, nullptr, k, lo, hi, sp, g0, part)
    if (arity == 16 && ncols == 16) KH_HA(16, 16);
    else if (arity == 16 && ncols == 8) KH_HA(16, 8);
    else if (arity == 8 && ncols == 16) KH_HA(8, 16);
    else if (arity == 8 && ncols == 8) KH_HA(8, 8);
    else {
        cudaFreeAsync(part, st);
        return gf_fail(GF_EINVAL, "fast array contraction needs arity / support 8 or 16");
    }
#undef KH_HA
    kh_pair_reduce_T<<<(ncols * arity + 255) / 256, 256, 0, st>>>(part, (double2 *)out, ctas, ncols, arity);
    GF_CUDA(cudaFreeAsync(part, st));
    GF_CUDA(cudaGetLastError());
    return GF_OK;
}

// ---------------------------------------------------------------------------
// handle
// ---------------------------------------------------------------------------
struct gf_hess_plan {
    int k, n, nlog, A, chunk;
    int64_t max_batch;
    u64 N;
    std::vector<HSlot> slots;
    std::vector<HSupport> sup;  // per slot (swapped support for swapped slots)
    std::vector<Mat4> G, Gt;
    bool have_gates = false;
    // pair CSR (reference _pair_csr)
    std::vector<int64_t> first_list, first_start, pair_second;
    int npairs = 0, R = 0;
    int64_t arrays_per_summand = 0;
    // device
    double2 *psis = nullptr, *phis = nullptr, *harr = nullptr, *harr2 = nullptr;
    double *partD = nullptr, *qD = nullptr, *partV = nullptr, *qV = nullptr;
    double2 *partP = nullptr, *qP = nullptr;
    int *d_lstart = nullptr, *d_lslots = nullptr, *d_swapped = nullptr, *d_rstart = nullptr, *d_rpairs = nullptr;
    int *d_sym = nullptr, *d_flip = nullptr;
    double *d_mult = nullptr;
    int64_t last_launches = 0;
};

static void hess_free(gf_hess_plan *h)
{
    void *ptrs[] = {h->psis, h->phis, h->harr, h->harr2, h->partD, h->qD, h->partV, h->qV, h->partP, h->qP,
                    h->d_lstart, h->d_lslots, h->d_swapped, h->d_rstart, h->d_rpairs, h->d_sym, h->d_flip,
                    h->d_mult};
    for (void *p : ptrs)
        if (p) cudaFree(p);
}


extern "C" int gf_hess_plan_create(gf_hess_plan **out, int k, int n_slots, const int32_t *t1, const int32_t *t2,
                                   const int32_t *logical, int n_logical, const int64_t *support, int arity,
                                   const int64_t *first_list, int64_t nfirst, const int64_t *first_start,
                                   const int64_t *pair_second, const double *pair_mult, const int64_t *pair_route,
                                   const int32_t *pair_sym, const int32_t *pair_flip, int64_t max_batch,
                                   int chunk_states)
{
    if (!out) return gf_fail(GF_EINVAL, "null plan pointer");
    *out = nullptr;
    if (k < 3 || k > 30) return gf_fail(GF_EINVAL, "qubit count %d out of range [3, 30]", k);
    if (n_slots < 1 || n_logical < 1 || max_batch < 1 || chunk_states < 1)
        return gf_fail(GF_EINVAL, "bad plan sizes");
    if (arity != 16 && arity != 8) return gf_fail(GF_EINVAL, "hole arity must be 16 (dense) or 8 (parity)");
    if (!t1 || !t2 || !logical || !support || (nfirst > 0 && (!first_list || !first_start)))
        return gf_fail(GF_EINVAL, "null argument");
    gf_hess_plan *h = new gf_hess_plan();
    h->k = k;
    h->n = n_slots;
    h->nlog = n_logical;
    h->A = arity;
    h->chunk = chunk_states;
    h->max_batch = max_batch;
    h->N = 1ull << k;
    h->R = n_logical * (n_logical + 1) / 2;
    static const int ws[4] = {0, 2, 1, 3};
    for (int s = 0; s < n_slots; ++s) {
        const int a = t1[s], b = t2[s];
        if (a == b || a < 0 || b < 0 || a >= k || b >= k || logical[s] < 0 || logical[s] >= n_logical) {
            delete h;
            return gf_fail(GF_EINVAL, "invalid slot %d: targets (%d, %d), logical %d", s, a, b, logical[s]);
        }
        HSlot si;
        si.swapped = a > b;
        si.lo = k - 1 - std::max(a, b);
        si.hi = k - 1 - std::min(a, b);
        si.logical = logical[s];
        si.sparse = false;
        h->slots.push_back(si);
        HSupport sp;
        for (int c = 0; c < arity; ++c) {
            const int64_t e = support[c];
            if (e < 0 || e > 15) {
                delete h;
                return gf_fail(GF_EINVAL, "support entry %lld outside [0, 15]", (long long)e);
            }
            int r = (int)(e / 4), cc = (int)(e % 4);
            if (si.swapped) {  // reference _swapped_support (kernels.py:568-571)
                r = ws[r];
                cc = ws[cc];
            }
            sp.row[c] = r;
            sp.col[c] = cc;
        }
        for (int c = arity; c < 16; ++c) sp.row[c] = sp.col[c] = 0;
        h->sup.push_back(sp);
    }
    // pair CSR
    const int64_t npairs = nfirst > 0 ? first_start[nfirst] : 0;
    h->npairs = (int)npairs;
    std::vector<int> rstart(h->R + 1, 0), rpairs, sym(std::max<int64_t>(1, npairs)), flip(std::max<int64_t>(1, npairs));
    std::vector<double> mult(std::max<int64_t>(1, npairs), 0.0);
    for (int64_t f = 0; f < nfirst; ++f) {
        const int64_t l = first_list[f];
        if (l < 0 || l >= n_slots || first_start[f + 1] <= first_start[f] || (f > 0 && first_list[f - 1] >= l)) {
            delete h;
            return gf_fail(GF_EINVAL, "bad pair CSR at first slot entry %lld", (long long)f);
        }
        int64_t prev = l;
        for (int64_t p = first_start[f]; p < first_start[f + 1]; ++p) {
            if (pair_second[p] <= prev || pair_second[p] >= n_slots || pair_route[p] < 0 || pair_route[p] >= h->R) {
                delete h;
                return gf_fail(GF_EINVAL, "bad pair CSR entry %lld", (long long)p);
            }
            prev = pair_second[p];
        }
        h->arrays_per_summand += pair_second[first_start[f + 1] - 1] - l - 1;
    }
    h->first_list.assign(first_list, first_list + nfirst);
    h->first_start.assign(first_start, first_start + nfirst + 1);
    h->pair_second.assign(pair_second, pair_second + npairs);
    for (int r = 0; r < h->R; ++r) {  // pairs of each route, in pair (CSR) order
        rstart[r] = (int)rpairs.size();
        for (int64_t p = 0; p < npairs; ++p)
            if (pair_route[p] == r) rpairs.push_back((int)p);
    }
    rstart[h->R] = (int)rpairs.size();
    for (int64_t p = 0; p < npairs; ++p) {
        mult[p] = pair_mult[p];
        sym[p] = pair_sym[p] != 0;
        flip[p] = pair_flip[p] != 0;
    }
    if (rpairs.empty()) rpairs.push_back(0);
    std::vector<int> lstart(n_logical + 1, 0), lslots, swp(n_slots);
    for (int l = 0; l < n_logical; ++l) {
        lstart[l] = (int)lslots.size();
        for (int s = 0; s < n_slots; ++s)
            if (logical[s] == l) lslots.push_back(s);
    }
    lstart[n_logical] = (int)lslots.size();
    for (int s = 0; s < n_slots; ++s) swp[s] = h->slots[s].swapped;
    // workspace
    const size_t vb = sizeof(double2) * h->N * (size_t)max_batch;
    const size_t ne = (size_t)arity * arity;
    cudaError_t e = cudaMalloc(&h->psis, vb * (n_slots + 1));
    if (e == cudaSuccess) e = cudaMalloc(&h->phis, vb * (n_slots + 1));
    if (e == cudaSuccess) e = cudaMalloc(&h->harr, vb * arity);
    if (e == cudaSuccess) e = cudaMalloc(&h->harr2, vb * arity);
    if (e == cudaSuccess) e = cudaMalloc(&h->partD, sizeof(double) * 32 * HMAXCTAS * max_batch);
    if (e == cudaSuccess) e = cudaMalloc(&h->qD, sizeof(double) * 32 * max_batch * n_slots);
    if (e == cudaSuccess) e = cudaMalloc(&h->partV, sizeof(double) * 2 * HMAXCTAS * max_batch);
    if (e == cudaSuccess) e = cudaMalloc(&h->qV, sizeof(double) * 2 * max_batch);
    if (e == cudaSuccess) e = cudaMalloc(&h->partP, sizeof(double2) * ne * HMAXCTAS * max_batch);
    if (e == cudaSuccess) e = cudaMalloc(&h->qP, sizeof(double2) * ne * max_batch * std::max<int64_t>(1, npairs));
    auto up = [&](int **dst, const std::vector<int> &v) {
        if (e == cudaSuccess) e = cudaMalloc(dst, sizeof(int) * v.size());
        if (e == cudaSuccess) e = cudaMemcpy(*dst, v.data(), sizeof(int) * v.size(), cudaMemcpyHostToDevice);
    };
    up(&h->d_lstart, lstart);
    up(&h->d_lslots, lslots.empty() ? std::vector<int>{0} : lslots);
    up(&h->d_swapped, swp);
    up(&h->d_rstart, rstart);
    up(&h->d_rpairs, rpairs);
    up(&h->d_sym, sym);
    up(&h->d_flip, flip);
    if (e == cudaSuccess) e = cudaMalloc(&h->d_mult, sizeof(double) * mult.size());
    if (e == cudaSuccess) e = cudaMemcpy(h->d_mult, mult.data(), sizeof(double) * mult.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        hess_free(h);
        delete h;
        cudaGetLastError();
        return gf_fail(e == cudaErrorMemoryAllocation ? GF_ENOMEM : GF_ECUDA, "hessian workspace: %s",
                       cudaGetErrorString(e));
    }
    *out = h;
    return GF_OK;
}

extern "C" int gf_hess_plan_set_gates(gf_hess_plan *h, const double *mats, int parity_mode)
{
    if (!h || !mats) return gf_fail(GF_EINVAL, "null argument");
    static const int s4[4] = {0, 2, 1, 3};
    static const int off[8] = {1, 2, 4, 7, 8, 11, 13, 14};
    h->G.resize(h->n);
    h->Gt.resize(h->n);
    for (int s = 0; s < h->n; ++s) {
        const double *m = mats + 32 * h->slots[s].logical;
        Mat4 g;
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) {
                const int e = h->slots[s].swapped ? 4 * s4[i] + s4[j] : 4 * i + j;
                g.m[4 * i + j] = make_double2(m[2 * e], m[2 * e + 1]);
            }
        bool zeros = true;
        for (int q : off) zeros = zeros && g.m[q].x == 0.0 && g.m[q].y == 0.0;
        h->slots[s].sparse = parity_mode && zeros;  // reference _Plan sparse flags (objective.py:188)
        h->G[s] = g;
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) h->Gt[s].m[4 * i + j] = g.m[4 * j + i];
    }
    h->have_gates = true;
    return GF_OK;
}

template <int A>
static int hess_pairs(gf_hess_plan *h, int64_t nvec, cudaStream_t st, int64_t &launches)
{
    constexpr int AS = A;  // support size == arity (DENSE_SUPPORT / PARITY_SUPPORT)
    const int K = h->k;
    const u64 N = h->N, units = N >> 2;
    const size_t lvl = (size_t)N * nvec;  // amplitudes per cache level
    const int ctas = grid_units(units, A);
    const dim3 grid(ctas, (unsigned)nvec);
    const size_t ne = (size_t)A * AS;
    int pidx = 0;
    for (size_t f = 0; f < h->first_list.size(); ++f) {
        const int l = (int)h->first_list[f];
        const int64_t p0 = h->first_start[f], p1 = h->first_start[f + 1];
        const int last = (int)h->pair_second[p1 - 1];
        const HSlot &sl = h->slots[l];
        kh_hole_apply<A><<<grid, HT, 0, st>>>(h->psis + (size_t)l * lvl, h->harr, K, sl.lo, sl.hi, h->sup[l]);
        ++launches;
        double2 *cur = h->harr, *nxt = h->harr2;
        int64_t pi = p0;
        for (int lp = l + 1; lp <= last; ++lp) {
            const HSlot &s2 = h->slots[lp];
            const bool contract = pi < p1 && h->pair_second[pi] == lp;
            const bool apply = lp < last;
            const double2 *bra = h->phis + (size_t)(h->n - lp - 1) * lvl;
            double2 *part = h->partP;
            const Mat4 &g = h->G[lp];
#define KH_PAIR(C, P, S) \
    kh_pair<A, AS, C, P, S><<<grid, HT, 0, st>>>(bra, cur, nxt, K, s2.lo, s2.hi, h->sup[lp], g, part)
            if (contract && apply) {
                if (s2.sparse) KH_PAIR(true, true, true); else KH_PAIR(true, true, false);
            } else if (contract) {
                KH_PAIR(true, false, false);
            } else if (s2.sparse) {
                kh_array_apply<A, true><<<grid, HT, 0, st>>>(cur, nxt, K, s2.lo, s2.hi, g);
            } else {
                kh_array_apply<A, false><<<grid, HT, 0, st>>>(cur, nxt, K, s2.lo, s2.hi, g);
            }
#undef KH_PAIR
            ++launches;
            if (contract) {
                const int64_t tot = nvec * (int64_t)ne;
                kh_pair_reduce<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
                    h->partP, h->qP + (size_t)pi * nvec * ne, nvec, ctas, (int)ne);
                ++launches;
                ++pi;
                ++pidx;
            }
            if (apply) std::swap(cur, nxt);
        }
    }
    (void)pidx;
    return GF_OK;
}

extern "C" int gf_hess_plan_eval(gf_hess_plan *h, int64_t nvec, const int64_t *basis, const double *weights,
                                 const void *phi0, double *out, int64_t *out_counts, void *stream)
{
    if (!h) return gf_fail(GF_EINVAL, "null plan");
    if (nvec < 1 || nvec > h->max_batch)
        return gf_fail(GF_EINVAL, "batch of %lld summands outside [1, %lld]", (long long)nvec, (long long)h->max_batch);
    if (!basis || !phi0 || !out) return gf_fail(GF_EINVAL, "null device buffer");
    if (!h->have_gates) return gf_fail(GF_EINVAL, "gates not set");
    cudaStream_t st = (cudaStream_t)stream;
    const int K = h->k, n = h->n;
    const u64 N = h->N, units = N >> 2;
    const size_t lvl = (size_t)N * nvec;
    int64_t launches = 0;
    {
        const u64 tot = lvl;
        kh_init<<<(unsigned)std::min<u64>((tot + 255) / 256, 148 * 16), 256, 0, st>>>(
            h->psis, h->phis, (const double2 *)phi0, basis, weights, N, nvec);
        ++launches;
    }
    // cached passes (objective.py:307-319)
    const u64 tu = units * (u64)nvec;
    const int ga = (int)std::min<u64>((tu + HT - 1) / HT, 148 * 16);
    for (int l = 0; l < n; ++l) {
        const HSlot &s = h->slots[l];
        if (s.sparse)
            kh_apply<true><<<ga, HT, 0, st>>>(h->psis + l * lvl, h->psis + (l + 1) * lvl, K, tu, s.lo, s.hi, h->G[l]);
        else
            kh_apply<false><<<ga, HT, 0, st>>>(h->psis + l * lvl, h->psis + (l + 1) * lvl, K, tu, s.lo, s.hi, h->G[l]);
        const int lb = n - 1 - l;  // phis[l+1] = G_{n-l-1}^T phis[l]
        const HSlot &sb = h->slots[lb];
        if (sb.sparse)
            kh_apply<true><<<ga, HT, 0, st>>>(h->phis + l * lvl, h->phis + (l + 1) * lvl, K, tu, sb.lo, sb.hi,
                                              h->Gt[lb]);
        else
            kh_apply<false><<<ga, HT, 0, st>>>(h->phis + l * lvl, h->phis + (l + 1) * lvl, K, tu, sb.lo, sb.hi,
                                               h->Gt[lb]);
        launches += 2;
    }
    // gradient holes D_l = hole(phis[n-l-1], psis[l]); value on slot 0's launch
    const int gh = grid_units(units, 1);
    for (int l = 0; l < n; ++l) {
        const HSlot &s = h->slots[l];
        const bool v = (l == 0);
        kh_hole<<<dim3(gh, (unsigned)nvec), HT, 0, st>>>(h->phis + (size_t)(n - l - 1) * lvl, h->psis + (size_t)l * lvl,
                                                         K, s.lo, s.hi, h->partD, v ? h->phis : nullptr,
                                                         v ? h->psis + (size_t)n * lvl : nullptr,
                                                         v ? h->partV : nullptr);
        kh_reduce<<<(unsigned)((nvec * 32 + 255) / 256), 256, 0, st>>>(h->partD, h->qD + (size_t)l * nvec * 32, nvec,
                                                                        gh, 32);
        launches += 2;
    }
    kh_reduce<<<(unsigned)((nvec * 2 + 255) / 256), 256, 0, st>>>(h->partV, h->qV, nvec, gh, 2);
    ++launches;
    int rc = h->A == 16 ? hess_pairs<16>(h, nvec, st, launches) : hess_pairs<8>(h, nvec, st, launches);
    if (rc) return rc;
    {
        const int64_t nchunks = (nvec + h->chunk - 1) / h->chunk;
        const int rec = 2 + 32 * h->nlog + 2 * h->R * h->A * h->A;
        const int64_t tot = nchunks * rec;
        kh_records<<<(unsigned)((tot * 32 + 255) / 256), 256, 0, st>>>(
            h->qD, h->qV, h->qP, nvec, n, h->nlog, h->d_lstart, h->d_lslots, h->d_swapped, h->d_rstart,
            h->d_rpairs, h->d_mult, h->d_sym, h->d_flip, h->A, h->R, h->chunk, out);
        ++launches;
    }
    GF_CUDA(cudaGetLastError());
    if (out_counts) {  // reference counter semantics (objective.py:65-73, 302-421)
        out_counts[0] += 2 * (int64_t)n * nvec;                  // gate applications
        out_counts[1] += h->arrays_per_summand * nvec;           // array gate applications
        out_counts[2] += (int64_t)h->first_list.size() * nvec;   // hole applications
        out_counts[3] += (int64_t)n * nvec;                      // hole contractions
        out_counts[4] += (int64_t)h->npairs * nvec;              // pair contractions
    }
    h->last_launches = launches;
    return GF_OK;
}

extern "C" int gf_hess_plan_slot_outputs(gf_hess_plan *h, int64_t nvec, double *d_dev, void *stream)
{
    if (!h || !d_dev || nvec < 1 || nvec > h->max_batch) return gf_fail(GF_EINVAL, "bad arguments");
    kh_slot_sums<<<(h->n * 32 + 255) / 256, 256, 0, (cudaStream_t)stream>>>(h->qD, nvec, h->n, d_dev);
    GF_CUDA(cudaGetLastError());
    return GF_OK;
}

extern "C" int64_t gf_hess_plan_last_launches(const gf_hess_plan *h) { return h ? h->last_launches : 0; }

extern "C" int gf_hess_plan_destroy(gf_hess_plan *h)
{
    if (!h) return GF_OK;
    hess_free(h);
    delete h;
    return GF_OK;
}
