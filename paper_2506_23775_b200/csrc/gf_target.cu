// gf_target.cu -- matrix-free target oracle on the GPU.
//
// phi0 = conj(exp(-iHt)|j>) is the input of every summand (reference
// objective.py:561-565).  The reference builds it on the CPU by a dense
// expm (models.py:305-319, <= 14 qubits) or a Lanczos subspace per state
// (models.py:322-384, ~370 ms per state at 16 qubits).  Here the
// hard-core-boson Hamiltonian (hopping bit-swaps + n_a n_b diagonal,
// reference models.py:37-45, 247-255) is applied matrix-free, optionally in
// the compressed parity sector, and exp(-iHt) is expanded in Chebyshev
// polynomials; one fused kernel per expansion order does
//   t_next = 2 Ht t_cur - t_prev,   acc += c_m t_next
// for a whole batch of columns.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "gf_common.cuh"
#include "gf_internal.h"

using namespace gf;

namespace {
constexpr int kMaxTerms = 96;

struct Terms {
    int n;
    int k;       // full-space qubits
    int sector;  // -1 full space, 0/1 compressed sector
    unsigned long long hop_mask[kMaxTerms];
    double hop_coef[kMaxTerms];
    int nhop;
    unsigned long long nn_mask[kMaxTerms];
    double nn_coef[kMaxTerms];
    int nnn;
};

__device__ __forceinline__ double2 happly(const double2 *__restrict__ v, u64 i, const Terms &T)
{
    // full-space index of the stored amplitude
    u64 x = (T.sector < 0) ? i : ((i << 1) | (u64)((__popcll(i) & 1) ^ T.sector));
    double d = 0.0;
    for (int t = 0; t < T.nnn; ++t)
        if ((x & T.nn_mask[t]) == T.nn_mask[t]) d += T.nn_coef[t];
    double2 acc = cscale(v[i], d);
    for (int t = 0; t < T.nhop; ++t) {
        u64 m = T.hop_mask[t];
        u64 b = x & m;
        if (b != 0 && b != m) {  // exactly one of the two bits set
            u64 y = x ^ m;
            u64 j = (T.sector < 0) ? y : (y >> 1);
            double2 w = v[j];
            acc.x = fma(T.hop_coef[t], w.x, acc.x);
            acc.y = fma(T.hop_coef[t], w.y, acc.y);
        }
    }
    return acc;
}

__global__ void __launch_bounds__(256) k_hamiltonian(const double2 *__restrict__ in, double2 *__restrict__ out,
                                                     int logN, u64 total, const Terms T)
{
    for (u64 g = (u64)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (u64)gridDim.x * blockDim.x) {
        u64 b = g >> logN, i = g & ((1ull << logN) - 1ull);
        out[g] = happly(in + (b << logN), i, T);
    }
}

__global__ void __launch_bounds__(256) k_cheb(const double2 *__restrict__ tcur, const double2 *__restrict__ tprev,
                                              double2 *__restrict__ tnext, double2 *__restrict__ acc, int logN,
                                              u64 total, const Terms T, double scale, double shift, double cre,
                                              double cim, int conj_out)
{
    for (u64 g = (u64)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (u64)gridDim.x * blockDim.x) {
        u64 b = g >> logN, i = g & ((1ull << logN) - 1ull);
        double2 h = happly(tcur + (b << logN), i, T);
        double2 c = tcur[g];
        h.x = fma(scale, h.x, shift * c.x);
        h.y = fma(scale, h.y, shift * c.y);
        if (tprev) {
            double2 p = tprev[g];
            h.x = 2.0 * h.x - p.x;
            h.y = 2.0 * h.y - p.y;
        }
        tnext[g] = h;
        if (acc) {
            double2 a = acc[g];
            // acc (+)= c * h, optionally stored conjugated-ready: conj_out
            // means acc holds conj(sum) so we add conj(c h).
            double2 ch = cmul(make_double2(cre, cim), h);
            if (conj_out) ch.y = -ch.y;
            a.x += ch.x;
            a.y += ch.y;
            acc[g] = a;
        }
    }
}

int make_terms(int k, const int32_t *ta, const int32_t *tb, const double *coef, const int32_t *hop, int nterms,
               int sector, Terms &T)
{
    if (nterms < 0 || nterms > kMaxTerms) return gf_fail(GF_EINVAL, "at most %d Hamiltonian terms", kMaxTerms);
    if (k < 2 || k > 40) return gf_fail(GF_EINVAL, "qubit count out of range");
    memset(&T, 0, sizeof T);
    T.k = k;
    T.sector = sector;
    for (int t = 0; t < nterms; ++t) {
        if (ta[t] < 0 || tb[t] < 0 || ta[t] >= k || tb[t] >= k || ta[t] == tb[t])
            return gf_fail(GF_EINVAL, "invalid term sites (%d, %d)", ta[t], tb[t]);
        u64 m = (1ull << (k - 1 - ta[t])) | (1ull << (k - 1 - tb[t]));
        if (hop[t]) {
            T.hop_mask[T.nhop] = m;
            T.hop_coef[T.nhop++] = coef[t];
        } else {
            T.nn_mask[T.nnn] = m;
            T.nn_coef[T.nnn++] = coef[t];
        }
    }
    T.n = nterms;
    return GF_OK;
}

int grid_for(u64 work) { return (int)std::max<u64>(1, std::min<u64>((work + 255) / 256, 148 * 16)); }
}  // namespace

extern "C" int gf_hamiltonian_apply(const void *in, void *out, int k, const int32_t *ta, const int32_t *tb,
                                    const double *coef, const int32_t *hop, int nterms, int64_t nvec, void *stream)
{
    if (!in || !out || in == out) return gf_fail(GF_EINVAL, "bad buffers (must be distinct, non-null)");
    Terms T;
    int rc = make_terms(k, ta, tb, coef, hop, nterms, -1, T);
    if (rc) return rc;
    u64 total = (1ull << k) * (u64)nvec;
    k_hamiltonian<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>((const double2 *)in, (double2 *)out, k, total, T);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return gf_fail(GF_ECUDA, "%s", cudaGetErrorString(e));
    return GF_OK;
}

// One Chebyshev order for a batch of nvec vectors of the stored space
// (sector -1: 2^k amplitudes, else 2^(k-1)).  H~ = scale*H + shift.
//   t_prev == NULL : t_next = H~ t_cur
//   otherwise      : t_next = 2 H~ t_cur - t_prev
//   acc (nullable) += c t_next   (conj(c t_next) when sector bit 8 set)
extern "C" int gf_cheb_step(const void *t_cur, const void *t_prev, void *t_next, void *acc, int k, const int32_t *ta,
                            const int32_t *tb, const double *coef, const int32_t *hop, int nterms, double scale,
                            double shift, double c_re, double c_im, int64_t nvec, int sector_flags, void *stream)
{
    if (!t_cur || !t_next || t_cur == t_next) return gf_fail(GF_EINVAL, "bad buffers");
    int sector = (sector_flags & 3) == 3 ? -1 : (sector_flags & 3);
    int conj_out = (sector_flags >> 8) & 1;
    Terms T;
    int rc = make_terms(k, ta, tb, coef, hop, nterms, sector, T);
    if (rc) return rc;
    int logN = sector < 0 ? k : k - 1;
    u64 total = (1ull << logN) * (u64)nvec;
    k_cheb<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>((const double2 *)t_cur, (const double2 *)t_prev,
                                                              (double2 *)t_next, (double2 *)acc, logN, total, T, scale,
                                                              shift, c_re, c_im, conj_out);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return gf_fail(GF_ECUDA, "%s", cudaGetErrorString(e));
    return GF_OK;
}

// ---------------------------------------------------------------------------
// Number-block target oracle.  Hopping terms conserve the particle number of
// each connected component of the hop graph (each spin chain for the
// Fermi-Hubbard models), so exp(-iHt)|j> lives in j's block: the states with
// the same particle count per component.  A block state is stored by its
// mixed-radix index x = sum_c r_c * stride_c, r_c the colex rank of the
// component's occupation pattern (positions p_0 < ... < p_{n-1},
// r = sum_t C(p_t, t+1)).  A hop between adjacent local positions i, i+1
// moves one particle without changing its index t among the particles, so
// the rank changes by +-C(i, t) (Pascal's rule): O(1) per term.
// ---------------------------------------------------------------------------
namespace {
constexpr int kMaxComp = 4, kMaxCompQ = 32, kMaxNbTerms = 96;

struct NbBlock {
    int ncomp;
    int k;                                 // full-space qubits
    int sector;                            // -1: dense rows of 2^k; 0/1: sector-compressed rows
    int L[kMaxComp], n[kMaxComp];          // component sizes / particle counts
    unsigned long long stride[kMaxComp];   // mixed-radix strides of the block index
    unsigned long long D;                  // block dimension
    unsigned char q[kMaxComp][kMaxCompQ];  // local position -> full qubit
    // terms: hop (comp, i, j: local positions, same component); nn (ca, ia, cb, ib)
    int nhop, nnn;
    unsigned char hc[kMaxNbTerms], hi[kMaxNbTerms], hj[kMaxNbTerms];
    double hcoef[kMaxNbTerms];
    unsigned char nca[kMaxNbTerms], nia[kMaxNbTerms], ncb[kMaxNbTerms], nib[kMaxNbTerms];
    double ncoef[kMaxNbTerms];
};

__constant__ unsigned long long c_binom[kMaxCompQ + 1][kMaxCompQ + 1];
// binomials indexed with thread-dependent (a, b): the kernels copy the table
// to shared memory, the constant cache would serialise divergent lookups
constexpr int kBin = kMaxCompQ + 1;
typedef unsigned long long BinTab[kBin];

__device__ __forceinline__ void load_binom(BinTab *s)
{
    for (int i = threadIdx.x; i < kBin * kBin; i += blockDim.x) s[i / kBin][i % kBin] = c_binom[i / kBin][i % kBin];
    __syncthreads();
}

// colex unrank: the n-particle pattern of rank r over positions [0, L)
// (binom[a][b] is zero for b > a, so the scan stops at the right position)
__device__ __forceinline__ unsigned unrank_colex(const BinTab *binom, unsigned long long r, int n, int L)
{
    unsigned pat = 0;
    int p = L - 1;
    for (int t = n; t >= 1; --t) {
        while (binom[p][t] > r) --p;
        pat |= 1u << p;
        r -= binom[p][t];
        --p;
    }
    return pat;
}

__device__ __forceinline__ unsigned long long rank_colex(const BinTab *binom, unsigned pat)
{
    unsigned long long r = 0;
    int t = 0;
    while (pat) {
        const int p = __ffs(pat) - 1;
        r += binom[p][++t];
        pat &= pat - 1;
    }
    return r;
}

// (H~ v)[x] for one block vector, H~ = scale * H + shift
__device__ __forceinline__ double2 nb_happly(const BinTab *binom, const double2 *__restrict__ v, unsigned long long x,
                                             const NbBlock &B)
{
    // block dimensions are < 2^32 (make_block), so the mixed-radix split
    // runs in 32-bit integer math
    unsigned pat[kMaxComp];
    unsigned long long r[kMaxComp];
    unsigned rem = (unsigned)x;
    for (int c = B.ncomp - 1; c >= 0; --c) {
        const unsigned rc = rem / (unsigned)B.stride[c];
        rem -= rc * (unsigned)B.stride[c];
        r[c] = rc;
        pat[c] = unrank_colex(binom, rc, B.n[c], B.L[c]);
    }
    double d = 0.0;
    for (int t = 0; t < B.nnn; ++t)
        if (((pat[B.nca[t]] >> B.nia[t]) & 1u) && ((pat[B.ncb[t]] >> B.nib[t]) & 1u)) d += B.ncoef[t];
    double2 acc = cscale(v[x], d);
    for (int t = 0; t < B.nhop; ++t) {
        const int c = B.hc[t], i = B.hi[t], j = B.hj[t];
        const unsigned bi = (pat[c] >> i) & 1u, bj = (pat[c] >> j) & 1u;
        if (bi == bj) continue;
        long long dr;
        if (j == i + 1) {
            // one particle crosses the adjacent pair; t = particles below i
            const int tt = __popc(pat[c] & ((1u << i) - 1u));
            const long long step = (long long)binom[i][tt];
            dr = bi ? step : -step;  // i -> i+1 raises the rank, i+1 -> i lowers it
        } else {
            dr = (long long)rank_colex(binom, pat[c] ^ ((1u << i) | (1u << j))) - (long long)r[c];
        }
        const double2 w = v[(unsigned long long)((long long)x + dr * (long long)B.stride[c])];
        acc.x = fma(B.hcoef[t], w.x, acc.x);
        acc.y = fma(B.hcoef[t], w.y, acc.y);
    }
    return acc;
}

__global__ void __launch_bounds__(256) k_nb_cheb(const double2 *__restrict__ tcur, const double2 *__restrict__ tprev,
                                                 double2 *__restrict__ tnext, double2 *__restrict__ acc,
                                                 unsigned long long total, const NbBlock B, double scale, double shift,
                                                 double cre, double cim)
{
    __shared__ BinTab binom[kBin];
    load_binom(binom);
    for (unsigned long long g = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; g < total;
         g += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long b = g / B.D, x = g - b * B.D;
        double2 h = nb_happly(binom, tcur + b * B.D, x, B);
        const double2 cc = tcur[g];
        h.x = fma(scale, h.x, shift * cc.x);
        h.y = fma(scale, h.y, shift * cc.y);
        if (tprev) {
            const double2 p = tprev[g];
            h.x = 2.0 * h.x - p.x;
            h.y = 2.0 * h.y - p.y;
        }
        tnext[g] = h;
        if (acc) {
            double2 a = acc[g];
            const double2 ch = cmul(make_double2(cre, cim), h);
            a.x += ch.x;
            a.y += ch.y;
            acc[g] = a;
        }
    }
}

// block vectors cols[colidx[b]] -> rows[rowidx[b]] (dense rows of 2^k, zeros
// outside the block; sector >= 0 stores rows compressed on qubit k-1,
// index = full >> 1).  Null index maps mean the identity.
__global__ void k_nb_scatter(const double2 *__restrict__ cols, const int64_t *__restrict__ colidx,
                             double2 *__restrict__ rows, const int64_t *__restrict__ rowidx, unsigned long long nrows,
                             unsigned long long N, const NbBlock B)
{
    __shared__ BinTab binom[kBin];
    load_binom(binom);
    const unsigned long long total = nrows * B.D;
    for (unsigned long long g = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; g < total;
         g += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long b = g / B.D, x = g - b * B.D;
        unsigned long long rem = x, full = 0;
        for (int c = B.ncomp - 1; c >= 0; --c) {
            const unsigned long long r = rem / B.stride[c];
            rem -= r * B.stride[c];
            unsigned pat = unrank_colex(binom, r, B.n[c], B.L[c]);
            while (pat) {
                const int pp = __ffs(pat) - 1;
                full |= 1ull << (B.k - 1 - B.q[c][pp]);
                pat &= pat - 1;
            }
        }
        const unsigned long long cb = colidx ? (unsigned long long)colidx[b] : b;
        const unsigned long long rb = rowidx ? (unsigned long long)rowidx[b] : b;
        rows[rb * N + (B.sector < 0 ? full : (full >> 1))] = cols[cb * B.D + x];
    }
}

// block index of full-space states: out[i] = x (the mixed-radix rank)
__global__ void k_nb_rank(const int64_t *__restrict__ js, int64_t *__restrict__ out, int64_t n, const NbBlock B)
{
    __shared__ BinTab binom[kBin];
    load_binom(binom);
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long j = (unsigned long long)js[g];
        unsigned long long x = 0;
        for (int c = 0; c < B.ncomp; ++c) {
            unsigned pat = 0;
            for (int i = 0; i < B.L[c]; ++i) pat |= (unsigned)((j >> (B.k - 1 - B.q[c][i])) & 1ull) << i;
            x += rank_colex(binom, pat) * B.stride[c];
        }
        out[g] = (int64_t)x;
    }
}

int make_block(const int32_t *desc, int ndesc, const int32_t *terms, const double *coef, int nterms, int sector,
               NbBlock &B)
{
    // desc: [k, ncomp, then per component: L, n, q_0 .. q_{L-1}]
    memset(&B, 0, sizeof B);
    if (ndesc < 2) return gf_fail(GF_EINVAL, "bad block descriptor");
    B.k = desc[0];
    B.ncomp = desc[1];
    B.sector = sector;
    if (B.ncomp < 1 || B.ncomp > kMaxComp || B.k < 2 || B.k > 40) return gf_fail(GF_EINVAL, "bad block descriptor");
    int pos = 2;
    unsigned long long D = 1;
    for (int c = 0; c < B.ncomp; ++c) {
        if (pos + 2 > ndesc) return gf_fail(GF_EINVAL, "truncated block descriptor");
        B.L[c] = desc[pos++];
        B.n[c] = desc[pos++];
        if (B.L[c] < 1 || B.L[c] > kMaxCompQ || B.n[c] < 0 || B.n[c] > B.L[c] || pos + B.L[c] > ndesc)
            return gf_fail(GF_EINVAL, "bad component");
        for (int i = 0; i < B.L[c]; ++i) B.q[c][i] = (unsigned char)desc[pos++];
        B.stride[c] = D;
        unsigned long long cnt = 1;
        for (int i = 0; i < B.n[c]; ++i) cnt = cnt * (B.L[c] - i) / (i + 1);
        D *= cnt;
    }
    if (D >= (1ull << 32)) return gf_fail(GF_EINVAL, "number block of dimension %llu too large", D);
    B.D = D;
    // terms: [kind(0 hop / 1 nn), ca, ia, cb, ib] x nterms
    for (int t = 0; t < nterms; ++t) {
        const int *r = terms + 5 * t;
        if (r[0] == 0) {
            if (B.nhop >= kMaxNbTerms || r[1] != r[3]) return gf_fail(GF_EINVAL, "hop term must stay in one component");
            int i = r[2], j = r[4];
            if (i > j) { int tmp = i; i = j; j = tmp; }
            B.hc[B.nhop] = (unsigned char)r[1];
            B.hi[B.nhop] = (unsigned char)i;
            B.hj[B.nhop] = (unsigned char)j;
            B.hcoef[B.nhop++] = coef[t];
        } else {
            if (B.nnn >= kMaxNbTerms) return gf_fail(GF_EINVAL, "too many terms");
            B.nca[B.nnn] = (unsigned char)r[1];
            B.nia[B.nnn] = (unsigned char)r[2];
            B.ncb[B.nnn] = (unsigned char)r[3];
            B.nib[B.nnn] = (unsigned char)r[4];
            B.ncoef[B.nnn++] = coef[t];
        }
    }
    return GF_OK;
}

bool g_binom_ready = false;
int ensure_binom()
{
    if (g_binom_ready) return GF_OK;
    unsigned long long h[kMaxCompQ + 1][kMaxCompQ + 1];
    memset(h, 0, sizeof h);
    for (int a = 0; a <= kMaxCompQ; ++a) {
        h[a][0] = 1;
        for (int b = 1; b <= a; ++b) h[a][b] = h[a - 1][b - 1] + (b <= a - 1 ? h[a - 1][b] : 0);
    }
    cudaError_t e = cudaMemcpyToSymbol(c_binom, h, sizeof h);
    if (e != cudaSuccess) return gf_fail(GF_ECUDA, "binomial table: %s", cudaGetErrorString(e));
    g_binom_ready = true;
    return GF_OK;
}
}  // namespace

// One Chebyshev order on nvec block vectors of one number block (see
// gf_cheb_step for the recurrence).  desc / terms describe the block
// (include/gatefit_b200.h).
extern "C" int gf_nb_cheb_step(const void *t_cur, const void *t_prev, void *t_next, void *acc, const int32_t *desc,
                               int ndesc, const int32_t *terms, const double *coef, int nterms, double scale,
                               double shift, double c_re, double c_im, int64_t nvec, void *stream)
{
    if (!t_cur || !t_next || nvec < 1) return gf_fail(GF_EINVAL, "bad buffers");
    int rc = ensure_binom();
    if (rc) return rc;
    NbBlock B;
    rc = make_block(desc, ndesc, terms, coef, nterms, -1, B);
    if (rc) return rc;
    const unsigned long long total = B.D * (unsigned long long)nvec;
    k_nb_cheb<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>((const double2 *)t_cur, (const double2 *)t_prev,
                                                                 (double2 *)t_next, (double2 *)acc, total, B, scale,
                                                                 shift, c_re, c_im);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return gf_fail(GF_ECUDA, "%s", cudaGetErrorString(e));
    return GF_OK;
}

// Scatter block vectors cols[colidx[b]] (D amplitudes each) into zeroed rows
// rows[rowidx[b]] of row_len amplitudes: dense (sector -1) or
// sector-compressed.  Null index maps mean the identity.
extern "C" int gf_nb_scatter(const void *cols, const int64_t *colidx, void *rows, const int64_t *rowidx, int64_t nrows,
                             int64_t row_len, const int32_t *desc, int ndesc, int sector, void *stream)
{
    if (!cols || !rows || nrows < 1) return gf_fail(GF_EINVAL, "bad buffers");
    int rc = ensure_binom();
    if (rc) return rc;
    NbBlock B;
    rc = make_block(desc, ndesc, nullptr, nullptr, 0, sector, B);
    if (rc) return rc;
    const unsigned long long total = B.D * (unsigned long long)nrows;
    k_nb_scatter<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>((const double2 *)cols, colidx, (double2 *)rows,
                                                                    rowidx, (unsigned long long)nrows,
                                                                    (unsigned long long)row_len, B);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return gf_fail(GF_ECUDA, "%s", cudaGetErrorString(e));
    return GF_OK;
}

// Block indices (mixed-radix colex ranks) of n full-space states that all
// lie in the block desc describes (device arrays).
extern "C" int gf_nb_rank(const int64_t *js, int64_t *out, int64_t n, const int32_t *desc, int ndesc, void *stream)
{
    if (!js || !out || n < 0) return gf_fail(GF_EINVAL, "bad buffers");
    if (n == 0) return GF_OK;
    int rc = ensure_binom();
    if (rc) return rc;
    NbBlock B;
    rc = make_block(desc, ndesc, nullptr, nullptr, 0, -1, B);
    if (rc) return rc;
    k_nb_rank<<<grid_for((unsigned long long)n), 256, 0, (cudaStream_t)stream>>>(js, out, n, B);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return gf_fail(GF_ECUDA, "%s", cudaGetErrorString(e));
    return GF_OK;
}

// Target rows from precomputed block matrices, no host round trip: row b gets
// mats[matoff[blk] + rank_of[j] * D + x] at full index full_of[stoff[blk] + x]
// for x < D (blk = block_of[j], D = blkdim[blk], j = js[b]); everything else
// in the row must already be zero.  Rows are dense (shift 0) or compressed on
// qubit k-1 (shift 1).
__global__ void k_nb_gather(const int64_t *__restrict__ js, const double2 *__restrict__ mats,
                            const int64_t *__restrict__ matoff, const int64_t *__restrict__ stoff,
                            const int32_t *__restrict__ blkdim, const int32_t *__restrict__ block_of,
                            const int32_t *__restrict__ rank_of, const int64_t *__restrict__ full_of, int shift,
                            double2 *__restrict__ out, int64_t row_len)
{
    const int64_t b = blockIdx.y;
    const int64_t j = js[b];
    const int blk = block_of[j];
    const int64_t D = blkdim[blk];
    const double2 *src = mats + matoff[blk] + (int64_t)rank_of[j] * D;
    const int64_t *dst = full_of + stoff[blk];
    double2 *row = out + b * row_len;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < D; x += (int64_t)gridDim.x * blockDim.x)
        row[dst[x] >> shift] = src[x];
}

extern "C" int gf_nb_gather(const int64_t *js, int64_t nrows, const void *mats, const int64_t *matoff,
                            const int64_t *stoff, const int32_t *blkdim, const int32_t *block_of,
                            const int32_t *rank_of, const int64_t *full_of, int64_t max_dim, int shift, void *out,
                            int64_t row_len, void *stream)
{
    if (!js || !mats || !out || nrows < 0 || max_dim < 1 || (shift != 0 && shift != 1) || nrows > 65535)
        return gf_fail(GF_EINVAL, "bad gather arguments");
    if (nrows == 0) return GF_OK;
    const unsigned gx = (unsigned)std::min<int64_t>((max_dim + 255) / 256, 64);
    k_nb_gather<<<dim3(gx, (unsigned)nrows), 256, 0, (cudaStream_t)stream>>>(
        js, (const double2 *)mats, matoff, stoff, blkdim, block_of, rank_of, full_of, shift, (double2 *)out, row_len);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return gf_fail(GF_ECUDA, "%s", cudaGetErrorString(e));
    return GF_OK;
}

// Block Hamiltonian as an ELL table (computed once per block; identical for
// every column): diag[x], cnt[x] valid hops, (nbr, coef) at t * D + x.
__global__ void k_nb_ell(const NbBlock B, double *__restrict__ diag, int *__restrict__ cnt, int *__restrict__ nbr,
                         double *__restrict__ hc, int nh)
{
    __shared__ BinTab binom[kBin];
    load_binom(binom);
    for (unsigned long long x = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; x < B.D;
         x += (unsigned long long)gridDim.x * blockDim.x) {
        unsigned pat[kMaxComp];
        unsigned long long r[kMaxComp];
        unsigned long long rem = x;
        for (int c = B.ncomp - 1; c >= 0; --c) {
            r[c] = rem / B.stride[c];
            rem -= r[c] * B.stride[c];
            pat[c] = unrank_colex(binom, r[c], B.n[c], B.L[c]);
        }
        double d = 0.0;
        for (int t = 0; t < B.nnn; ++t)
            if (((pat[B.nca[t]] >> B.nia[t]) & 1u) && ((pat[B.ncb[t]] >> B.nib[t]) & 1u)) d += B.ncoef[t];
        diag[x] = d;
        int k = 0;
        for (int t = 0; t < B.nhop; ++t) {
            const int c = B.hc[t], i = B.hi[t], j = B.hj[t];
            const unsigned bi = (pat[c] >> i) & 1u, bj = (pat[c] >> j) & 1u;
            if (bi == bj) continue;
            long long dr;
            if (j == i + 1) {
                const long long step = (long long)binom[i][__popc(pat[c] & ((1u << i) - 1u))];
                dr = bi ? step : -step;
            } else {
                dr = (long long)rank_colex(binom, pat[c] ^ ((1u << i) | (1u << j))) - (long long)r[c];
            }
            nbr[k * B.D + x] = (int)((long long)x + dr * (long long)B.stride[c]);
            hc[k * B.D + x] = B.hcoef[t];
            ++k;
        }
        cnt[x] = k;
    }
}

// Whole block matrix in one launch: CTA b runs every Chebyshev order of
// column e_b on chip.  cur and prev live in shared memory (neighbours read
// cur; each thread overwrites only its own prev entries with next, then the
// two buffers swap roles); the ELL Hamiltonian and the accumulator row out[b]
// stay L2-resident.  Row b of the result = sum_m c_m T_m(H~) e_b.  The hop
// terms are summed in term order after the diagonal, exactly as nb_happly.
__global__ void __launch_bounds__(1024) k_nb_series(double2 *__restrict__ out, const double2 *__restrict__ coefs,
                                                    int norder, long long D, const double *__restrict__ diag,
                                                    const int *__restrict__ cnt, const int *__restrict__ nbr,
                                                    const double *__restrict__ hc, int nh, double scale, double shift)
{
    extern __shared__ double2 nb_smem[];
    const long long b = blockIdx.x;
    double2 *cur = nb_smem, *prev = nb_smem + D;
    double2 *row = out + b * D;
    const double2 c0 = coefs[0];
    // the thread's entries of the result row accumulate in registers (D <= 6400,
    // at least 32 threads per 32 entries: at most NB_ACC entries per thread)
    constexpr int NB_ACC = 8;
    double2 acc[NB_ACC];
#pragma unroll
    for (int i = 0; i < NB_ACC; ++i) acc[i] = make_double2(0.0, 0.0);
    {
        int i = 0;
        for (long long x = threadIdx.x; x < D; x += blockDim.x, ++i) {
            const double v = (x == b) ? 1.0 : 0.0;
            cur[x] = make_double2(v, 0.0);
            const double2 a0 = make_double2(c0.x * v, c0.y * v);
#pragma unroll
            for (int q = 0; q < NB_ACC; ++q)
                if (q == i) acc[q] = a0;
        }
    }
    __syncthreads();
    for (int m = 1; m <= norder; ++m) {
        const double2 cm = coefs[m];
        int i = 0;
        for (long long x = threadIdx.x; x < D; x += blockDim.x, ++i) {
            const double2 cc = cur[x];
            double2 h = cscale(cc, diag[x]);
            const int k = cnt[x];
            for (int t = 0; t < k; ++t) {
                const double w = hc[t * D + x];
                const double2 v = cur[nbr[t * D + x]];
                h.x = fma(w, v.x, h.x);
                h.y = fma(w, v.y, h.y);
            }
            h.x = fma(scale, h.x, shift * cc.x);
            h.y = fma(scale, h.y, shift * cc.y);
            if (m > 1) {
                const double2 p = prev[x];
                h.x = 2.0 * h.x - p.x;
                h.y = 2.0 * h.y - p.y;
            }
            prev[x] = h;
            const double2 ch = cmul(cm, h);
#pragma unroll
            for (int q = 0; q < NB_ACC; ++q)
                if (q == i) {
                    acc[q].x += ch.x;
                    acc[q].y += ch.y;
                }
        }
        __syncthreads();
        double2 *t = cur;
        cur = prev;
        prev = t;
    }
    {
        int i = 0;
        for (long long x = threadIdx.x; x < D; x += blockDim.x, ++i) {
#pragma unroll
            for (int q = 0; q < NB_ACC; ++q)
                if (q == i) row[x] = acc[q];
        }
    }
}

// Block matrix (rows conj(U e_b) in block coordinates when coefs are the
// conjugated series coefficients) for one number block, D <= 6400.
// coefs: device array of norder + 1 complex coefficients.  work: device
// scratch of at least D * (16 + 12 * nhop) bytes for the ELL Hamiltonian.
extern "C" int gf_nb_block_matrix(void *out, const int32_t *desc, int ndesc, const int32_t *terms, const double *coef,
                                  int nterms, const void *coefs, int norder, double scale, double shift, void *work,
                                  void *stream)
{
    if (!out || !coefs || !work || norder < 1) return gf_fail(GF_EINVAL, "bad block-matrix arguments");
    int rc = ensure_binom();
    if (rc) return rc;
    NbBlock B;
    rc = make_block(desc, ndesc, terms, coef, nterms, -1, B);
    if (rc) return rc;
    const size_t smem = 2 * sizeof(double2) * (size_t)B.D;
    if (smem > 200 * 1024) return gf_fail(GF_EINVAL, "block dimension %llu too large for on-chip series", B.D);
    static bool attr = false;
    if (!attr) {
        cudaError_t ae = cudaFuncSetAttribute(k_nb_series, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (ae != cudaSuccess) return gf_fail(GF_ECUDA, "k_nb_series smem attribute: %s", cudaGetErrorString(ae));
        attr = true;
    }
    const int nh = std::max(1, B.nhop);
    char *w = (char *)work;
    double *diag = (double *)w;
    double *hc = diag + B.D;
    int *nbr = (int *)(hc + B.D * nh);
    int *cnt = nbr + B.D * nh;
    cudaStream_t st = (cudaStream_t)stream;
    k_nb_ell<<<grid_for(B.D), 256, 0, st>>>(B, diag, cnt, nbr, hc, nh);
    const int nt = (int)std::min<unsigned long long>(1024, (B.D + 31) / 32 * 32);
    k_nb_series<<<(unsigned)B.D, nt, smem, st>>>((double2 *)out, (const double2 *)coefs, norder, (long long)B.D, diag,
                                                 cnt, nbr, hc, nh, scale, shift);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return gf_fail(GF_ECUDA, "%s", cudaGetErrorString(e));
    return GF_OK;
}
