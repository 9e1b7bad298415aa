// gf_ops.cu -- kernel-level C-ABI operations (reference kernels.py public ops),
// parity-sector index maps, translation-orbit folding, error plumbing.
#include <cuda_runtime.h>
#include <cstdint>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "gf_common.cuh"
#include "gf_internal.h"

using namespace gf;

static thread_local char g_err[1024] = "";

void gf_set_error(const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

int gf_fail(int code, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

extern "C" const char *gf_last_error(void) { return g_err; }
extern "C" int gf_abi_version(void) { return 100; }

#define GF_CUDA(call)                                                                               \
    do {                                                                                            \
        cudaError_t _e = (call);                                                                    \
        if (_e != cudaSuccess)                                                                      \
            return gf_fail(_e == cudaErrorMemoryAllocation ? GF_ENOMEM : GF_ECUDA, "%s:%d %s (%s)", \
                           __FILE__, __LINE__, cudaGetErrorName(_e), cudaGetErrorString(_e));       \
    } while (0)

namespace {

struct Norm {
    int q1, q2;
    bool swapped;
    int lo, hi;
};

int normalise(int k, int t1, int t2, Norm &n)
{
    if (t1 == t2) return gf_fail(GF_EINVAL, "gate targets must be distinct");
    if (t1 < 0 || t2 < 0 || t1 >= k || t2 >= k)
        return gf_fail(GF_EINVAL, "targets (%d, %d) out of range for %d qubits", t1, t2, k);
    n.swapped = t1 > t2;
    n.q1 = std::min(t1, t2);
    n.q2 = std::max(t1, t2);
    n.lo = k - 1 - n.q2;
    n.hi = k - 1 - n.q1;
    return GF_OK;
}

Mat4 load_mat(const double *m, bool swapped)
{
    static const int s[4] = {0, 2, 1, 3};
    Mat4 r;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            int e = swapped ? 4 * s[i] + s[j] : 4 * i + j;
            r.m[4 * i + j] = make_double2(m[2 * e], m[2 * e + 1]);
        }
    return r;
}

int grid_for(unsigned long long work, int threads, int cap = 148 * 16)
{
    unsigned long long b = (work + threads - 1) / threads;
    return (int)std::max<unsigned long long>(1, std::min<unsigned long long>(b, (unsigned long long)cap));
}

struct Support {
    int n;
    int row[16], col[16];
};

int make_support(const int64_t *support, int arity, bool swapped, Support &s)
{
    static const int ws[4] = {0, 2, 1, 3};
    if (arity < 1 || arity > 16) return gf_fail(GF_EINVAL, "support size %d outside [1, 16]", arity);
    s.n = arity;
    for (int a = 0; a < arity; ++a) {
        int64_t e = support ? support[a] : a;
        if (e < 0 || e > 15) return gf_fail(GF_EINVAL, "support entry %lld outside [0, 15]", (long long)e);
        int r = (int)(e / 4), c = (int)(e % 4);
        if (swapped) {
            r = ws[r];
            c = ws[c];
        }
        s.row[a] = r;
        s.col[a] = c;
    }
    return GF_OK;
}

}  // namespace

namespace gf {

// K1: standalone streaming gate application (batched over vectors).
// Each thread handles UNROLL tuples per trip with all loads issued before the
// FMAs, for memory-level parallelism; in-place safe (disjoint tuples).
template <bool SPARSE, int UNROLL>
__global__ void __launch_bounds__(256) k_apply2q(const double2 *__restrict__ in, double2 *out, int logN,
                                                 unsigned long long total, int lo, int hi, const Mat4 g)
{
    const int logU = logN - 2;
    const u64 umask = (1ull << logU) - 1ull;
    const u64 ol = 1ull << lo, oh = 1ull << hi;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 t0 = (u64)blockIdx.x * blockDim.x + threadIdx.x; t0 < total; t0 += stride * UNROLL) {
        double2 x[UNROLL][4];
        u64 base[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            u64 t = t0 + (u64)u * stride;
            if (t < total) {
                u64 v = t >> logU, r = t & umask;
                base[u] = (v << logN) | ins0(ins0(r, lo), hi);
                x[u][0] = in[base[u]];
                x[u][1] = in[base[u] + ol];
                x[u][2] = in[base[u] + oh];
                x[u][3] = in[base[u] + ol + oh];
            }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            u64 t = t0 + (u64)u * stride;
            if (t < total) {
                double2 y[4];
                mv4<SPARSE>(g, x[u], y);
                out[base[u]] = y[0];
                out[base[u] + ol] = y[1];
                out[base[u] + oh] = y[2];
                out[base[u] + ol + oh] = y[3];
            }
        }
    }
}

// 256-bit global accesses (LDG/STG.E.ENL2.256 on sm_100a)
__device__ __forceinline__ void ld256(const double2 *p, double2 &a, double2 &b)
{
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y) : "l"(p));
}
__device__ __forceinline__ void st256(double2 *p, double2 a, double2 b)
{
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y)
                 : "memory");
}

// K1 for a low target on bit 0: the two amplitudes of each pair are adjacent
// and 32 B aligned, so each thread moves them with one 256-bit access instead
// of two 128-bit ones that each fill half of every 32 B sector.  (Measured:
// pairs on bit 0 ran at 5.2-5.7 TB/s against ~6.2 TB/s elsewhere.)
template <bool SPARSE, int UNROLL>
__global__ void __launch_bounds__(256) k_apply2q_lo0(const double2 *__restrict__ in, double2 *out, int logN,
                                                     unsigned long long total, int hi, const Mat4 g)
{
    const int logU = logN - 2;
    const u64 umask = (1ull << logU) - 1ull;
    const u64 oh = 1ull << hi;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 t0 = (u64)blockIdx.x * blockDim.x + threadIdx.x; t0 < total; t0 += stride * UNROLL) {
        double2 x[UNROLL][4];
        u64 base[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const u64 t = t0 + (u64)u * stride;
            if (t < total) {
                const u64 v = t >> logU, r = t & umask;
                base[u] = (v << logN) | ins0(ins0(r, 0), hi);
                ld256(in + base[u], x[u][0], x[u][1]);
                ld256(in + base[u] + oh, x[u][2], x[u][3]);
            }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const u64 t = t0 + (u64)u * stride;
            if (t < total) {
                double2 y[4];
                mv4<SPARSE>(g, x[u], y);
                st256(out + base[u], y[0], y[1]);
                st256(out + base[u] + oh, y[2], y[3]);
            }
        }
    }
}

// the parity-controlled 1q gate on bit 0: one 256-bit access per pair
template <int UNROLL>
__global__ void __launch_bounds__(256) k_apply_c1q_lo0(const double2 *__restrict__ in, double2 *out, int logN,
                                                       unsigned long long total, int sector, const Mat4 g)
{
    const int logU = logN - 1;
    const u64 umask = (1ull << logU) - 1ull;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 t0 = (u64)blockIdx.x * blockDim.x + threadIdx.x; t0 < total; t0 += stride * UNROLL) {
        double2 x[UNROLL][2];
        u64 base[UNROLL];
        int P[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const u64 t = t0 + (u64)u * stride;
            if (t < total) {
                const u64 v = t >> logU, r = ins0(t & umask, 0);
                P[u] = (__popcll(r) & 1) ^ sector;
                base[u] = (v << logN) | r;
                ld256(in + base[u], x[u][0], x[u][1]);
            }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const u64 t = t0 + (u64)u * stride;
            if (t < total) {
                double2 y[2];
                mv2(g, P[u], x[u], y);
                st256(out + base[u], y[0], y[1]);
            }
        }
    }
}

// K1 for targets above bit 0: tuples t and t + 1 (t even) have bases b and
// b + 1, so a thread applies the gate to both and moves each amplitude pair
// of the two tuples with one 256-bit access.
template <bool SPARSE, int UNROLL>
__global__ void __launch_bounds__(256) k_apply2q_x2(const double2 *__restrict__ in, double2 *out, int logN,
                                                    unsigned long long npairs, int lo, int hi, const Mat4 g)
{
    const int logU = logN - 2;
    const u64 umask = (1ull << logU) - 1ull;
    const u64 ol = 1ull << lo, oh = 1ull << hi;
    const u64 off[4] = {0ull, ol, oh, ol + oh};
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 p0 = (u64)blockIdx.x * blockDim.x + threadIdx.x; p0 < npairs; p0 += stride * UNROLL) {
        double2 xe[UNROLL][4], xo[UNROLL][4];
        u64 base[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const u64 pp = p0 + (u64)u * stride;
            if (pp < npairs) {
                const u64 t = 2 * pp, v = t >> logU, r = t & umask;
                base[u] = (v << logN) | ins0(ins0(r, lo), hi);
#pragma unroll
                for (int i = 0; i < 4; ++i) ld256(in + base[u] + off[i], xe[u][i], xo[u][i]);
            }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const u64 pp = p0 + (u64)u * stride;
            if (pp < npairs) {
                double2 ye[4], yo[4];
                mv4<SPARSE>(g, xe[u], ye);
                mv4<SPARSE>(g, xo[u], yo);
#pragma unroll
                for (int i = 0; i < 4; ++i) st256(out + base[u] + off[i], ye[i], yo[i]);
            }
        }
    }
}

// the parity-controlled 1q gate above bit 0: pairs r and r + 1 (r even) per
// thread, opposite parities, 256-bit accesses
template <int UNROLL>
__global__ void __launch_bounds__(256) k_apply_c1q_x2(const double2 *__restrict__ in, double2 *out, int logN,
                                                      unsigned long long npairs, int pa, int sector, const Mat4 g)
{
    const int logU = logN - 1;
    const u64 umask = (1ull << logU) - 1ull;
    const u64 o = 1ull << pa;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 p0 = (u64)blockIdx.x * blockDim.x + threadIdx.x; p0 < npairs; p0 += stride * UNROLL) {
        double2 xe[UNROLL][2], xo[UNROLL][2];
        u64 base[UNROLL];
        int P[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const u64 pp = p0 + (u64)u * stride;
            if (pp < npairs) {
                const u64 t = 2 * pp, v = t >> logU, r = ins0(t & umask, pa);
                P[u] = (__popcll(r) & 1) ^ sector;
                base[u] = (v << logN) | r;
                ld256(in + base[u], xe[u][0], xo[u][0]);
                ld256(in + base[u] + o, xe[u][1], xo[u][1]);
            }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const u64 pp = p0 + (u64)u * stride;
            if (pp < npairs) {
                double2 ye[2], yo[2];
                mv2(g, P[u], xe[u], ye);
                mv2(g, P[u] ^ 1, xo[u], yo);
                st256(out + base[u], ye[0], yo[0]);
                st256(out + base[u] + o, ye[1], yo[1]);
            }
        }
    }
}

// parity-controlled one-qubit gate of the compressed sector space
template <int UNROLL>
__global__ void __launch_bounds__(256) k_apply_c1q(const double2 *__restrict__ in, double2 *out, int logN,
                                                   unsigned long long total, int pa, int sector, const Mat4 g)
{
    const int logU = logN - 1;
    const u64 umask = (1ull << logU) - 1ull;
    const u64 o = 1ull << pa;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 t0 = (u64)blockIdx.x * blockDim.x + threadIdx.x; t0 < total; t0 += stride * UNROLL) {
        double2 x[UNROLL][2];
        u64 base[UNROLL];
        int P[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            u64 t = t0 + (u64)u * stride;
            if (t < total) {
                u64 v = t >> logU, r = ins0(t & umask, pa);
                P[u] = (__popcll(r) & 1) ^ sector;
                base[u] = (v << logN) | r;
                x[u][0] = in[base[u]];
                x[u][1] = in[base[u] + o];
            }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            u64 t = t0 + (u64)u * stride;
            if (t < total) {
                double2 y[2];
                mv2(g, P[u], x[u], y);
                out[base[u]] = y[0];
                out[base[u] + o] = y[1];
            }
        }
    }
}

// hole contraction summed over nvec vector pairs -> per-CTA partials
__global__ void __launch_bounds__(256) k_hole(const double2 *__restrict__ bra, const double2 *__restrict__ ket,
                                              int logN, unsigned long long total, int lo, int hi, double *part)
{
    const int logU = logN - 2;
    const u64 umask = (1ull << logU) - 1ull;
    const u64 ol = 1ull << lo, oh = 1ull << hi;
    double acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = 0.0;
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (u64)gridDim.x * blockDim.x) {
        u64 v = t >> logU, r = t & umask;
        u64 b = (v << logN) | ins0(ins0(r, lo), hi);
        double2 y[4] = {bra[b], bra[b + ol], bra[b + oh], bra[b + ol + oh]};
        double2 x[4] = {ket[b], ket[b + ol], ket[b + oh], ket[b + ol + oh]};
        hole_acc(acc, y, x);
    }
    __shared__ double red[256];
    double s = block_reduce32(acc, red);
    if (threadIdx.x < 32) part[(u64)blockIdx.x * 32 + threadIdx.x] = s;
}

// final: sum partials over CTAs (ascending) and un-swap into caller orientation
__global__ void k_hole_final(const double *part, int nparts, int swapped, double *out)
{
    int q = threadIdx.x;  // 32 threads
    if (q >= 32) return;
    int e = q >> 1, ri = q & 1, i = e >> 2, j = e & 3;
    if (swapped) {
        i = (i == 1) ? 2 : (i == 2 ? 1 : i);
        j = (j == 1) ? 2 : (j == 2 ? 1 : j);
    }
    int src = 2 * (4 * i + j) + ri;
    double acc = 0.0;
    for (int c = 0; c < nparts; ++c) acc += part[c * 32 + src];
    out[q] = acc;
}

struct SupportDev {
    int n;
    int row[16], col[16];
};

__global__ void k_hole_apply(const double2 *__restrict__ psi, double2 *out, int logN, int lo, int hi,
                             const SupportDev sup)
{
    const u64 total = (1ull << logN) * (u64)sup.n;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (u64)gridDim.x * blockDim.x) {
        u64 phys = i / sup.n;
        int a = (int)(i - phys * sup.n);
        int tb = (int)(((phys >> hi) & 1) * 2 + ((phys >> lo) & 1));
        double2 v = make_double2(0.0, 0.0);
        if (tb == sup.row[a]) {
            int c = sup.col[a];
            u64 src = (phys & ~((1ull << hi) | (1ull << lo))) | ((u64)(c >> 1) << hi) | ((u64)(c & 1) << lo);
            v = psi[src];
        }
        out[i] = v;
    }
}

template <bool SPARSE>
__global__ void k_array_apply(const double2 *__restrict__ in, double2 *__restrict__ out, int logN, int A, int lo,
                              int hi, const Mat4 g)
{
    const u64 units = 1ull << (logN - 2);
    const u64 total = units * (u64)A;
    const u64 ol = 1ull << lo, oh = 1ull << hi;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (u64)gridDim.x * blockDim.x) {
        u64 t = i / A;
        int a = (int)(i - t * A);
        u64 b = ins0(ins0(t, lo), hi);
        u64 r[4] = {b, b + ol, b + oh, b + ol + oh};
        double2 x[4], y[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) x[q] = in[r[q] * A + a];
        mv4<SPARSE>(g, x, y);
#pragma unroll
        for (int q = 0; q < 4; ++q) out[r[q] * A + a] = y[q];
    }
}

// outT[c][a] partial sums; thread (c, a) = threadIdx.x < ncols*A
__global__ void k_hole_array(const double2 *__restrict__ bra, const double2 *__restrict__ arr, int logN, int A,
                             int lo, int hi, const SupportDev sup, double2 *part)
{
    const int ncols = sup.n;
    const int me = threadIdx.x;
    const bool active = me < ncols * A;
    const int c = active ? me / A : 0, a = active ? me % A : 0;
    const u64 units = 1ull << (logN - 2);
    const u64 ol = 1ull << lo, oh = 1ull << hi;
    const int ri = sup.row[c], ci = sup.col[c];
    const u64 offr = ((ri >> 1) ? oh : 0) + ((ri & 1) ? ol : 0);
    const u64 offc = ((ci >> 1) ? oh : 0) + ((ci & 1) ? ol : 0);
    double2 acc = make_double2(0.0, 0.0);
    if (active) {
        for (u64 t = blockIdx.x; t < units; t += gridDim.x) {
            u64 b = ins0(ins0(t, lo), hi);
            acc = cfma(bra[b + offr], arr[(b + offc) * A + a], acc);
        }
        part[(u64)blockIdx.x * ncols * A + me] = acc;
    }
}

// reduce [nparts][ncols*A] -> out[a][c] (transpose to the reference's B[a, c])
__global__ void k_hole_array_final(const double2 *part, int nparts, int ncols, int A, double2 *out)
{
    int me = blockIdx.x * blockDim.x + threadIdx.x;
    if (me >= ncols * A) return;
    int c = me / A, a = me % A;
    double2 acc = make_double2(0.0, 0.0);
    for (int p = 0; p < nparts; ++p) acc = cadd(acc, part[(u64)p * ncols * A + me]);
    out[a * ncols + c] = acc;
}

// ---- sector index maps ---------------------------------------------------
__global__ void k_unrank(const int64_t *idx, int64_t m, int sector, int64_t *out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        u64 v = (u64)idx[i];
        out[i] = (int64_t)((v << 1) | (u64)((__popcll(v) & 1) ^ sector));
    }
}

__global__ void k_rank(const int64_t *x, int64_t m, int64_t *out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = x[i] >> 1;
}

// 2-site translation of both spin chains: within each L-bit chain field
// (qubit 0 of the chain = field MSB) qubit s -> s+2 mod L is a rotate right
// by 2.  Up chain = high L bits, down chain = low L bits.
__device__ __forceinline__ u64 rotr2(u64 f, int L)
{
    const u64 mask = (1ull << L) - 1ull;
    return ((f >> 2) | ((f & 3ull) << (L - 2))) & mask;
}

__device__ __forceinline__ u64 shift2(u64 x, int L)
{
    const u64 mask = (1ull << L) - 1ull;
    return (rotr2(x >> L, L) << L) | rotr2(x & mask, L);
}

__device__ __forceinline__ void canon(u64 x, int L, u64 &rep, int &size)
{
    const int period = (L % 2 == 0) ? L / 2 : L;
    u64 best = x, y = x;
    int sz = period;
    for (int s = 1; s < period; ++s) {
        y = shift2(y, L);
        if (y == x && sz == period) sz = s;
        best = y < best ? y : best;
    }
    rep = best;
    size = sz;
}

__global__ void k_orbit_canon(const int64_t *x, int64_t m, int L, int64_t *rep, int64_t *size)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        u64 r;
        int s;
        canon((u64)x[i], L, r, s);
        rep[i] = (int64_t)r;
        size[i] = s;
    }
}

__global__ void k_orbit_mark(int64_t i0, int64_t m, int L, int sector, int32_t *mark)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        u64 v = (u64)(i0 + i);
        u64 x = (v << 1) | (u64)((__popcll(v) & 1) ^ sector);
        u64 r;
        int s;
        canon(x, L, r, s);
        mark[i] = (r == x) ? s : 0;
    }
}

}  // namespace gf

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------

static int log2_exact(int k) { return k; }

extern "C" int gf_apply_gate(const void *in, void *out, int k, int t1, int t2, const double *mat, int parity_sparse,
                             int64_t nvec, void *stream)
{
    if (!in || !out || !mat) return gf_fail(GF_EINVAL, "null argument");
    if (k < 2 || k > 40) return gf_fail(GF_EINVAL, "qubit count %d out of range", k);
    if (nvec < 1) return gf_fail(GF_EINVAL, "nvec must be >= 1");
    Norm nm;
    int rc = normalise(k, t1, t2, nm);
    if (rc) return rc;
    Mat4 g = load_mat(mat, nm.swapped);
    unsigned long long total = (1ull << (k - 2)) * (unsigned long long)nvec;
    int grid = grid_for(total, 256 * 2, 148 * 32);
    cudaStream_t st = (cudaStream_t)stream;
    // 256-bit accesses need 32 B aligned vectors (a view at an odd amplitude
    // offset falls back to the 128-bit kernel)
    const bool a32 = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 31u) == 0;
    if (nm.lo == 0 && a32) {
        if (parity_sparse)
            k_apply2q_lo0<true, 2><<<grid, 256, 0, st>>>((const double2 *)in, (double2 *)out, log2_exact(k), total,
                                                         nm.hi, g);
        else
            k_apply2q_lo0<false, 2><<<grid, 256, 0, st>>>((const double2 *)in, (double2 *)out, log2_exact(k), total,
                                                          nm.hi, g);
    } else if (a32 && k >= 3 && !(nm.lo == 1 && nm.hi == 2)) {
        // (bits 1 and 2: a thread's four 256-bit accesses would be one 128 B
        // run with lanes 128 B apart -- measured 4.8 TB/s; the plain kernel
        // keeps ~6.2)
        const unsigned long long np = total / 2;  // 2^(k-2) tuples per vector: even
        const int grid2 = grid_for(np, 256 * 2, 148 * 32);
        if (parity_sparse)
            k_apply2q_x2<true, 2><<<grid2, 256, 0, st>>>((const double2 *)in, (double2 *)out, log2_exact(k), np,
                                                         nm.lo, nm.hi, g);
        else
            k_apply2q_x2<false, 2><<<grid2, 256, 0, st>>>((const double2 *)in, (double2 *)out, log2_exact(k), np,
                                                          nm.lo, nm.hi, g);
    } else if (parity_sparse)
        k_apply2q<true, 2><<<grid, 256, 0, st>>>((const double2 *)in, (double2 *)out, log2_exact(k), total, nm.lo,
                                                 nm.hi, g);
    else
        k_apply2q<false, 2><<<grid, 256, 0, st>>>((const double2 *)in, (double2 *)out, log2_exact(k), total, nm.lo,
                                                  nm.hi, g);
    GF_CUDA(cudaGetLastError());
    return GF_OK;
}

extern "C" int gf_apply_gate_sector_c1q(const void *in, void *out, int k_full, int a, int sector, const double *mat,
                                        int64_t nvec, void *stream)
{
    if (!in || !out || !mat) return gf_fail(GF_EINVAL, "null argument");
    if (k_full < 3 || k_full > 41) return gf_fail(GF_EINVAL, "qubit count out of range");
    if (a < 0 || a >= k_full - 1) return gf_fail(GF_EINVAL, "target %d must be an explicit qubit", a);
    if (sector != 0 && sector != 1) return gf_fail(GF_EINVAL, "sector must be 0 or 1");
    Mat4 g = load_mat(mat, false);
    static const int off[8] = {1, 2, 4, 7, 8, 11, 13, 14};
    for (int e : off)
        if (g.m[e].x != 0.0 || g.m[e].y != 0.0) return gf_fail(GF_EINVAL, "gate is not parity-conserving");
    int K = k_full - 1;
    int pa = K - 1 - a;
    unsigned long long total = (1ull << (K - 1)) * (unsigned long long)nvec;
    int grid = grid_for(total, 256 * 2, 148 * 32);
    const bool a32 = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 31u) == 0;
    if (pa == 0 && a32)
        k_apply_c1q_lo0<2><<<grid, 256, 0, (cudaStream_t)stream>>>((const double2 *)in, (double2 *)out, K, total,
                                                                   sector, g);
    else if (a32 && K >= 3)
        k_apply_c1q_x2<2><<<grid_for(total / 2, 256 * 2, 148 * 32), 256, 0, (cudaStream_t)stream>>>(
            (const double2 *)in, (double2 *)out, K, total / 2, pa, sector, g);
    else
        k_apply_c1q<2><<<grid, 256, 0, (cudaStream_t)stream>>>((const double2 *)in, (double2 *)out, K, total, pa,
                                                               sector, g);
    GF_CUDA(cudaGetLastError());
    return GF_OK;
}

// Generic one-qubit gate (north-star item 1).  The reference absorbs 1q gates
// into its 2q gates; the engine-side kernels are the
// parity-controlled 1q kernels with both 2x2 blocks set to the same matrix,
// so every amplitude pair gets g whatever its parity (same 256-bit paths).
extern "C" int gf_apply_gate_1q(const void *in, void *out, int k, int q, const double *mat, int64_t nvec,
                                void *stream)
{
    if (!in || !out || !mat) return gf_fail(GF_EINVAL, "null argument");
    if (k < 1 || k > 40 || nvec < 1) return gf_fail(GF_EINVAL, "bad sizes");
    if (q < 0 || q >= k) return gf_fail(GF_EINVAL, "target %d out of range for %d qubits", q, k);
    Mat4 g;
    for (int e = 0; e < 16; ++e) g.m[e] = make_double2(0.0, 0.0);
    const double2 a = make_double2(mat[0], mat[1]), b = make_double2(mat[2], mat[3]);
    const double2 c = make_double2(mat[4], mat[5]), d = make_double2(mat[6], mat[7]);
    g.m[0] = a; g.m[3] = b; g.m[12] = c; g.m[15] = d;   // parity-0 block
    g.m[5] = a; g.m[6] = b; g.m[9] = c; g.m[10] = d;    // parity-1 block
    const int pa = k - 1 - q;
    const unsigned long long total = (1ull << (k - 1)) * (unsigned long long)nvec;
    const int grid = grid_for(total, 256 * 2, 148 * 32);
    cudaStream_t st = (cudaStream_t)stream;
    const bool a32 = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 31u) == 0;
    if (pa == 0 && a32)
        k_apply_c1q_lo0<2><<<grid, 256, 0, st>>>((const double2 *)in, (double2 *)out, k, total, 0, g);
    else if (a32 && k >= 2 && total >= 2)
        k_apply_c1q_x2<2><<<grid_for(total / 2, 256 * 2, 148 * 32), 256, 0, st>>>(
            (const double2 *)in, (double2 *)out, k, total / 2, pa, 0, g);
    else
        k_apply_c1q<2><<<grid, 256, 0, st>>>((const double2 *)in, (double2 *)out, k, total, pa, 0, g);
    GF_CUDA(cudaGetLastError());
    return GF_OK;
}

extern "C" int gf_hole_contract(const void *bra, const void *ket, int k, int t1, int t2, int64_t nvec, void *out_dev,
                                void *stream)
{
    if (!bra || !ket || !out_dev) return gf_fail(GF_EINVAL, "null argument");
    if (k < 2 || k > 40 || nvec < 1) return gf_fail(GF_EINVAL, "bad sizes");
    Norm nm;
    int rc = normalise(k, t1, t2, nm);
    if (rc) return rc;
    unsigned long long total = (1ull << (k - 2)) * (unsigned long long)nvec;
    int grid = grid_for(total, 256 * 4, 148 * 8);
    double *part = nullptr;
    cudaStream_t st = (cudaStream_t)stream;
    GF_CUDA(cudaMallocAsync((void **)&part, sizeof(double) * 32 * grid, st));
    k_hole<<<grid, 256, 0, st>>>((const double2 *)bra, (const double2 *)ket, k, total, nm.lo, nm.hi, part);
    k_hole_final<<<1, 32, 0, st>>>(part, grid, nm.swapped, (double *)out_dev);
    GF_CUDA(cudaFreeAsync(part, st));
    GF_CUDA(cudaGetLastError());
    return GF_OK;
}

extern "C" int gf_hole_apply(const void *psi, void *out, int k, int t1, int t2, const int64_t *support, int arity,
                             void *stream)
{
    if (!psi || !out) return gf_fail(GF_EINVAL, "null argument");
    if (k < 2 || k > 36) return gf_fail(GF_EINVAL, "qubit count out of range");
    Norm nm;
    int rc = normalise(k, t1, t2, nm);
    if (rc) return rc;
    Support s;
    rc = make_support(support, arity, nm.swapped, s);
    if (rc) return rc;
    if (arity == 16 || arity == 8) return gf_fast_hole_apply(psi, out, k, nm.lo, nm.hi, s.row, s.col, arity, stream);
    SupportDev sd;
    sd.n = s.n;
    memcpy(sd.row, s.row, sizeof sd.row);
    memcpy(sd.col, s.col, sizeof sd.col);
    unsigned long long total = (1ull << k) * (unsigned long long)arity;
    k_hole_apply<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>((const double2 *)psi, (double2 *)out, k,
                                                                        nm.lo, nm.hi, sd);
    GF_CUDA(cudaGetLastError());
    return GF_OK;
}

extern "C" int gf_apply_gate_to_array(const void *in, void *out, int k, int arity, int t1, int t2, const double *mat,
                                      int parity_sparse, void *stream)
{
    if (!in || !out || !mat) return gf_fail(GF_EINVAL, "null argument");
    if (in == out) return gf_fail(GF_EINVAL, "output buffer must not alias the input array");
    if (k < 2 || k > 36 || arity < 1) return gf_fail(GF_EINVAL, "bad sizes");
    Norm nm;
    int rc = normalise(k, t1, t2, nm);
    if (rc) return rc;
    Mat4 g = load_mat(mat, nm.swapped);
    if (arity == 16 || arity == 8) return gf_fast_array_apply(in, out, k, arity, nm.lo, nm.hi, g, parity_sparse, stream);
    unsigned long long total = (1ull << (k - 2)) * (unsigned long long)arity;
    cudaStream_t st = (cudaStream_t)stream;
    if (parity_sparse)
        k_array_apply<true><<<grid_for(total, 256), 256, 0, st>>>((const double2 *)in, (double2 *)out, k, arity,
                                                                  nm.lo, nm.hi, g);
    else
        k_array_apply<false><<<grid_for(total, 256), 256, 0, st>>>((const double2 *)in, (double2 *)out, k, arity,
                                                                   nm.lo, nm.hi, g);
    GF_CUDA(cudaGetLastError());
    return GF_OK;
}

extern "C" int gf_hole_contract_array(const void *bra, const void *arr, int k, int arity, int t1, int t2,
                                      const int64_t *support, int ncols, void *out_dev, void *stream)
{
    if (!bra || !arr || !out_dev) return gf_fail(GF_EINVAL, "null argument");
    if (k < 2 || k > 36 || arity < 1 || arity > 16) return gf_fail(GF_EINVAL, "bad sizes");
    Norm nm;
    int rc = normalise(k, t1, t2, nm);
    if (rc) return rc;
    Support s;
    rc = make_support(support, ncols, nm.swapped, s);
    if (rc) return rc;
    if ((arity == 16 || arity == 8) && (ncols == 16 || ncols == 8))
        return gf_fast_hole_array(bra, arr, k, arity, nm.lo, nm.hi, s.row, s.col, ncols, out_dev, stream);
    SupportDev sd;
    sd.n = s.n;
    memcpy(sd.row, s.row, sizeof sd.row);
    memcpy(sd.col, s.col, sizeof sd.col);
    const int threads = ((ncols * arity + 31) / 32) * 32;
    const unsigned long long units = 1ull << (k - 2);
    int grid = (int)std::min<unsigned long long>(units, 148 * 8);
    cudaStream_t st = (cudaStream_t)stream;
    double2 *part = nullptr;
    GF_CUDA(cudaMallocAsync((void **)&part, sizeof(double2) * (size_t)grid * ncols * arity, st));
    k_hole_array<<<grid, threads, 0, st>>>((const double2 *)bra, (const double2 *)arr, k, arity, nm.lo, nm.hi, sd,
                                          part);
    k_hole_array_final<<<(ncols * arity + 255) / 256, 256, 0, st>>>(part, grid, ncols, arity, (double2 *)out_dev);
    GF_CUDA(cudaFreeAsync(part, st));
    GF_CUDA(cudaGetLastError());
    return GF_OK;
}

__global__ void k_count_nonfinite(const double *x, int64_t n, unsigned long long *bad)
{
    unsigned long long local = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        local += isfinite(x[i]) ? 0ull : 1ull;
    if (local) atomicAdd(bad, local);  // integer count: order-independent
}

// Synchronous: GF_ENONFINITE if any of the n doubles is NaN / Inf (the
// reference raises FloatingPointError on non-finite results,
// objective.py:575-578, optimizer.py:147-149).
extern "C" int gf_check_finite(const double *x, int64_t n, void *stream)
{
    if (n < 0 || (n > 0 && !x)) return gf_fail(GF_EINVAL, "bad arguments");
    if (n == 0) return GF_OK;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long *bad = nullptr, host = 0;
    GF_CUDA(cudaMallocAsync((void **)&bad, sizeof *bad, st));
    GF_CUDA(cudaMemsetAsync(bad, 0, sizeof *bad, st));
    k_count_nonfinite<<<grid_for((unsigned long long)n, 256), 256, 0, st>>>(x, n, bad);
    GF_CUDA(cudaMemcpyAsync(&host, bad, sizeof host, cudaMemcpyDeviceToHost, st));
    GF_CUDA(cudaFreeAsync(bad, st));
    GF_CUDA(cudaStreamSynchronize(st));
    if (host) return gf_fail(GF_ENONFINITE, "%llu non-finite values in %lld engine outputs", host, (long long)n);
    return GF_OK;
}

extern "C" int gf_sector_unrank(const int64_t *idx, int64_t m, int sector, int64_t *out, void *stream)
{
    if (m < 0 || (m > 0 && (!idx || !out))) return gf_fail(GF_EINVAL, "bad arguments");
    if (sector != 0 && sector != 1) return gf_fail(GF_EINVAL, "sector must be 0 or 1");
    if (m == 0) return GF_OK;
    k_unrank<<<grid_for(m, 256), 256, 0, (cudaStream_t)stream>>>(idx, m, sector, out);
    GF_CUDA(cudaGetLastError());
    return GF_OK;
}

extern "C" int gf_sector_rank(const int64_t *x, int64_t m, int64_t *out, void *stream)
{
    if (m < 0 || (m > 0 && (!x || !out))) return gf_fail(GF_EINVAL, "bad arguments");
    if (m == 0) return GF_OK;
    k_rank<<<grid_for(m, 256), 256, 0, (cudaStream_t)stream>>>(x, m, out);
    GF_CUDA(cudaGetLastError());
    return GF_OK;
}

extern "C" int gf_orbit_canon(const int64_t *x, int64_t m, int L, int64_t *rep, int64_t *size, void *stream)
{
    if (m < 0 || L < 2 || L > 31) return gf_fail(GF_EINVAL, "bad arguments");
    if (m == 0) return GF_OK;
    k_orbit_canon<<<grid_for(m, 256), 256, 0, (cudaStream_t)stream>>>(x, m, L, rep, size);
    GF_CUDA(cudaGetLastError());
    return GF_OK;
}

extern "C" int gf_sector_orbit_mark(int64_t i0, int64_t m, int L, int sector, int32_t *mark, void *stream)
{
    if (m < 0 || L < 2 || L > 31 || (sector != 0 && sector != 1)) return gf_fail(GF_EINVAL, "bad arguments");
    if (m == 0) return GF_OK;
    k_orbit_mark<<<grid_for(m, 256), 256, 0, (cudaStream_t)stream>>>(i0, m, L, sector, mark);
    GF_CUDA(cudaGetLastError());
    return GF_OK;
}

// ---------------------------------------------------------------------------
// Peak microbenchmarks (measurement helpers for bench.py's roofline: neither
// MEASURED_PEAKS.json nor the profiling recipe states an FP64 peak).
// 8 independent accumulator chains per thread, back to back.
// ---------------------------------------------------------------------------
namespace gf {
__global__ void __launch_bounds__(256) k_peak_dmma(double *sink, int iters)
{
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - blockIdx.x * 1e-9;
    double c[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+d"(c[j][0]), "+d"(c[j][1])
                : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
    if (s == -1.0) sink[0] = s;
}

__global__ void __launch_bounds__(256) k_peak_dfma(double *sink, int iters)
{
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - blockIdx.x * 1e-9;
    double c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j] = fma(c[j], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j];
    if (s == -1.0) sink[0] = s;
}
__global__ void __launch_bounds__(256) k_peak_mixed(double *sink, int iters)
{
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - blockIdx.x * 1e-9;
    double c[8][2], d[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = d[j] = j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+d"(c[j][0]), "+d"(c[j][1])
                : "d"(a), "d"(b));
            d[j] = fma(d[j], a, b);
            d[j] = fma(d[j], b, a);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + d[j];
    if (s == -1.0) sink[0] = s;
}
}  // namespace gf

// which: 0 = DMMA m8n8k4 (512 flop per warp instruction), 1 = DFMA (2 flop
// per thread instruction).  Returns the flop count of the launch in *flops.
extern "C" int gf_peak_fp64(int which, int blocks, int iters, double *sink_dev, double *flops, void *stream)
{
    if (!sink_dev || !flops || blocks < 1 || iters < 1) return gf_fail(GF_EINVAL, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    if (which == 0) {
        k_peak_dmma<<<blocks, 256, 0, st>>>(sink_dev, iters);
        *flops = (double)blocks * 8 /*warps*/ * iters * 8 * 512.0;
    } else if (which == 1) {
        k_peak_dfma<<<blocks, 256, 0, st>>>(sink_dev, iters);
        *flops = (double)blocks * 256 * iters * 8 * 2.0;
    } else {
        // 2: DMMA and DFMA interleaved (are the FP64 tensor and FMA pipes independent?)
        k_peak_mixed<<<blocks, 256, 0, st>>>(sink_dev, iters);
        *flops = (double)blocks * 8 * iters * 8 * 512.0 + (double)blocks * 256 * iters * 8 * 4.0;
    }
    GF_CUDA(cudaGetLastError());
    return GF_OK;
}

// ---------------------------------------------------------------------------
// Minimal device-memory helpers so a binding without a tensor library (e.g.
// a ctypes stub inside the reference's objective.py) can drive the ABI.
// ---------------------------------------------------------------------------
extern "C" int gf_set_device(int device)
{
    GF_CUDA(cudaSetDevice(device));
    return GF_OK;
}

extern "C" int gf_malloc(void **ptr, int64_t bytes)
{
    if (!ptr || bytes < 0) return gf_fail(GF_EINVAL, "bad arguments");
    *ptr = nullptr;
    if (bytes == 0) return GF_OK;
    GF_CUDA(cudaMalloc(ptr, (size_t)bytes));
    return GF_OK;
}

extern "C" int gf_free(void *ptr)
{
    if (ptr) GF_CUDA(cudaFree(ptr));
    return GF_OK;
}

extern "C" int gf_memcpy(void *dst, const void *src, int64_t bytes, int kind, void *stream)
{
    // kind: 0 host->device, 1 device->host, 2 device->device
    if (bytes < 0 || kind < 0 || kind > 2) return gf_fail(GF_EINVAL, "bad arguments");
    if (bytes == 0) return GF_OK;
    const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice
                                       : (kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice);
    GF_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, k, (cudaStream_t)stream));
    return GF_OK;
}

extern "C" int gf_stream_sync(void *stream)
{
    GF_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    return GF_OK;
}
