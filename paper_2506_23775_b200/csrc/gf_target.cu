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
