// gf_common.cuh -- shared device helpers for the sm_100a contraction engine.
//
// State vectors are complex128 stored as double2 (re, im), length N = 2^K with
// qubit 0 the MOST significant bit (reference kernels.py:6-10).  A two-qubit
// slot acts on bit positions hi > lo (hi = K-1-q1, lo = K-1-q2 for q1 < q2);
// its gate index is 2*bit(hi) + bit(lo) (reference kernels.py:17-19).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gf {

typedef unsigned long long u64;

struct Mat4 {  // row-major 4x4 complex, m[4*i + j]
    double2 m[16];
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b)
{
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// c + a*b
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c)
{
    c.x = fma(a.x, b.x, c.x);
    c.x = fma(-a.y, b.y, c.x);
    c.y = fma(a.x, b.y, c.y);
    c.y = fma(a.y, b.x, c.y);
    return c;
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 czero() { return make_double2(0.0, 0.0); }

// insert a zero bit at position b
__device__ __forceinline__ u64 ins0(u64 t, int b)
{
    u64 low = t & ((1ull << b) - 1ull);
    return ((t >> b) << (b + 1)) | low;
}

// y = M x for a 4-vector (dense), SPARSE skips the 8 structural zeros of a
// parity-conserving gate (reference kernels.py:283-322).
template <bool SPARSE>
__device__ __forceinline__ void mv4(const Mat4 &M, const double2 x[4], double2 y[4])
{
    if (SPARSE) {
        y[0] = cfma(M.m[3], x[3], cmul(M.m[0], x[0]));
        y[1] = cfma(M.m[6], x[2], cmul(M.m[5], x[1]));
        y[2] = cfma(M.m[10], x[2], cmul(M.m[9], x[1]));
        y[3] = cfma(M.m[15], x[3], cmul(M.m[12], x[0]));
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            double2 s = cmul(M.m[4 * i], x[0]);
            s = cfma(M.m[4 * i + 1], x[1], s);
            s = cfma(M.m[4 * i + 2], x[2], s);
            s = cfma(M.m[4 * i + 3], x[3], s);
            y[i] = s;
        }
    }
}

// y += M x
template <bool SPARSE>
__device__ __forceinline__ void mv4_acc(const Mat4 &M, const double2 x[4], double2 y[4])
{
    if (SPARSE) {
        y[0] = cfma(M.m[3], x[3], cfma(M.m[0], x[0], y[0]));
        y[1] = cfma(M.m[6], x[2], cfma(M.m[5], x[1], y[1]));
        y[2] = cfma(M.m[10], x[2], cfma(M.m[9], x[1], y[2]));
        y[3] = cfma(M.m[15], x[3], cfma(M.m[12], x[0], y[3]));
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            double2 s = y[i];
#pragma unroll
            for (int j = 0; j < 4; ++j) s = cfma(M.m[4 * i + j], x[j], s);
            y[i] = s;
        }
    }
}

// Hole accumulator: acc[2*(4i+j)] (+1 for imag) += bra[i] * ket[j]
// (reference kernels.py:208-242; bra is NOT conjugated).
__device__ __forceinline__ void hole_acc(double acc[32], const double2 bra[4], const double2 ket[4])
{
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            double2 a = make_double2(acc[2 * (4 * i + j)], acc[2 * (4 * i + j) + 1]);
            a = cfma(bra[i], ket[j], a);
            acc[2 * (4 * i + j)] = a.x;
            acc[2 * (4 * i + j) + 1] = a.y;
        }
}

// Parity-controlled 1q block of a 4x4 gate: P=0 -> rows/cols {0,3},
// P=1 -> {1,2} (sector compression of the implicit last qubit).
__device__ __forceinline__ void sub2(const Mat4 &M, int P, double2 &a, double2 &b, double2 &c, double2 &d)
{
    // [a b; c d] = M[[i0,i1],[i0,i1]]
    if (P == 0) {
        a = M.m[0]; b = M.m[3]; c = M.m[12]; d = M.m[15];
    } else {
        a = M.m[5]; b = M.m[6]; c = M.m[9]; d = M.m[10];
    }
}

__device__ __forceinline__ void mv2(const Mat4 &M, int P, const double2 x[2], double2 y[2])
{
    double2 a, b, c, d;
    sub2(M, P, a, b, c, d);
    y[0] = cfma(b, x[1], cmul(a, x[0]));
    y[1] = cfma(d, x[1], cmul(c, x[0]));
}

__device__ __forceinline__ void mv2_acc(const Mat4 &M, int P, const double2 x[2], double2 y[2])
{
    double2 a, b, c, d;
    sub2(M, P, a, b, c, d);
    y[0] = cfma(b, x[1], cfma(a, x[0], y[0]));
    y[1] = cfma(d, x[1], cfma(c, x[0], y[1]));
}

// hole accumulation of a controlled-1q pair: entries {0,3}x{0,3} when P=0,
// {1,2}x{1,2} when P=1 (disjoint entry sets, so both are kept statically).
__device__ __forceinline__ void hole_acc2(double acc[32], int P, const double2 bra[2], const double2 ket[2])
{
    double2 p00 = cmul(bra[0], ket[0]), p01 = cmul(bra[0], ket[1]);
    double2 p10 = cmul(bra[1], ket[0]), p11 = cmul(bra[1], ket[1]);
    double e = (P == 0) ? 1.0 : 0.0, o = 1.0 - e;
    // P=0 entries: 0, 3, 12, 15
    acc[0] = fma(e, p00.x, acc[0]);   acc[1] = fma(e, p00.y, acc[1]);
    acc[6] = fma(e, p01.x, acc[6]);   acc[7] = fma(e, p01.y, acc[7]);
    acc[24] = fma(e, p10.x, acc[24]); acc[25] = fma(e, p10.y, acc[25]);
    acc[30] = fma(e, p11.x, acc[30]); acc[31] = fma(e, p11.y, acc[31]);
    // P=1 entries: 5, 6, 9, 10
    acc[10] = fma(o, p00.x, acc[10]); acc[11] = fma(o, p00.y, acc[11]);
    acc[12] = fma(o, p01.x, acc[12]); acc[13] = fma(o, p01.y, acc[13]);
    acc[18] = fma(o, p10.x, acc[18]); acc[19] = fma(o, p10.y, acc[19]);
    acc[20] = fma(o, p11.x, acc[20]); acc[21] = fma(o, p11.y, acc[21]);
}

// Warp reduce-scatter of 32 doubles: afterwards lane l holds sum over lanes
// of acc[l] in acc[0].  31 shuffles instead of 5*32 for a full all-reduce.
__device__ __forceinline__ double warp_reduce_scatter32(double acc[32])
{
    const unsigned lane = threadIdx.x & 31u;
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const bool upper = (lane & s) != 0;
#pragma unroll
        for (int i = 0; i < s; ++i) {
            double send = upper ? acc[i] : acc[i + s];
            double keep = upper ? acc[i + s] : acc[i];
            acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
        }
    }
    return acc[0];
}

// Deterministic block reduction of a 32-double accumulator; thread 0..31 of
// warp 0 get the block total of entry lane.  smem must hold nwarps*32 doubles.
__device__ __forceinline__ double block_reduce32(double acc[32], double *smem)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double v = warp_reduce_scatter32(acc);
    smem[warp * 32 + lane] = v;
    __syncthreads();
    double tot = 0.0;
    if (warp == 0)
        for (int w = 0; w < nw; ++w) tot += smem[w * 32 + lane];
    __syncthreads();
    return tot;
}

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace gf
