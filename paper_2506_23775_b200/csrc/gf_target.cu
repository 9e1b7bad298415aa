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

__device__ __forceinline__ unsigned long long binom(int a, int b)
{
    return (b < 0 || b > a) ? 0ull : c_binom[a][b];
}

// colex unrank: the n-particle pattern of rank r over positions [0, L)
__device__ __forceinline__ unsigned unrank_colex(unsigned long long r, int n, int L)
{
    unsigned pat = 0;
    int p = L - 1;
    for (int t = n; t >= 1; --t) {
        while (binom(p, t) > r) --p;
        pat |= 1u << p;
        r -= binom(p, t);
        --p;
    }
    return pat;
}

__device__ __forceinline__ unsigned long long rank_colex(unsigned pat)
{
    unsigned long long r = 0;
    int t = 0;
    while (pat) {
        const int p = __ffs(pat) - 1;
        r += binom(p, ++t);
        pat &= pat - 1;
    }
    return r;
}

// (H~ v)[x] for one block vector, H~ = scale * H + shift
__device__ __forceinline__ double2 nb_happly(const double2 *__restrict__ v, unsigned long long x, const NbBlock &B)
{
    unsigned pat[kMaxComp];
    unsigned long long r[kMaxComp];
    unsigned long long rem = x;
    for (int c = B.ncomp - 1; c >= 0; --c) {
        r[c] = rem / B.stride[c];
        rem -= r[c] * B.stride[c];
        pat[c] = unrank_colex(r[c], B.n[c], B.L[c]);
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
            const long long step = (long long)binom(i, tt);
            dr = bi ? step : -step;  // i -> i+1 raises the rank, i+1 -> i lowers it
        } else {
            dr = (long long)rank_colex(pat[c] ^ ((1u << i) | (1u << j))) - (long long)r[c];
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
    for (unsigned long long g = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; g < total;
         g += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long b = g / B.D, x = g - b * B.D;
        double2 h = nb_happly(tcur + b * B.D, x, B);
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
    const unsigned long long total = nrows * B.D;
    for (unsigned long long g = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; g < total;
         g += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long b = g / B.D, x = g - b * B.D;
        unsigned long long rem = x, full = 0;
        for (int c = B.ncomp - 1; c >= 0; --c) {
            const unsigned long long r = rem / B.stride[c];
            rem -= r * B.stride[c];
            unsigned pat = unrank_colex(r, B.n[c], B.L[c]);
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
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long j = (unsigned long long)js[g];
        unsigned long long x = 0;
        for (int c = 0; c < B.ncomp; ++c) {
            unsigned pat = 0;
            for (int i = 0; i < B.L[c]; ++i) pat |= (unsigned)((j >> (B.k - 1 - B.q[c][i])) & 1ull) << i;
            x += rank_colex(pat) * B.stride[c];
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
