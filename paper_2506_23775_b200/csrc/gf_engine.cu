// gf_engine.cu -- batched basis-sum engine: fused forward / reverse / ascending
// sweeps over a batch of summands, deterministic reductions, C-ABI plan.
//
// Reference semantics (gatefit, arXiv 2506.23775):
//   forward      psi_{l+1} = G_l psi_l                         objective.py:310-313
//   backward     phi_m = G_{n-m}^T phi_{m-1}, phi_0 = conj(U|j>)  objective.py:314-317
//   gradient     D_l = hole(phi_{n-l-1}, psi_l)                objective.py:333-335
//   HVP          ascending / descending recursions             objective.py:461-482
// The B200 engine replaces the 2(n+1)-vector pass cache with a reversible
// 3-vector schedule (SURVEY 7 "hard parts" 2): psi is uncomputed with G^dag,
// the bra is propagated with G^T on the way down and recovered with conj(G)
// on the way up.
//
// Default engine (k_fused): a sweep is a few *passes* planned on the host
// (plan_passes: exact beam over local-bit sets when affordable).  One launch
// per pass stages 2^m-amplitude tiles of psi / bra / chi (or v) in shared
// memory -- one CTA per tile, two CTAs per SM -- and runs all of the pass's
// slots on them: FP64 tensor-core (DMMA m8n8k4) gate applications and hole
// contractions, per-slot partials written per CTA and summed in CTA order by
// k_reduce_ctas.  Parity-sector plans run the same passes as FP64 FMAs on
// two-amplitude units instead (run_units, PM_UNIT: the block-diagonal slots of
// a sector waste half of every DMMA).  The streaming engine (k_sweep, one
// launch per slot) serves tiny state spaces and GF_ENGINE=stream.
//
// Compile-time switches (measured defaults): GF_FUSED_GH -- fused gate + hole
// phase in the ascending passes; GF_FUSED_BLOCK -- its groups per load batch;
// GF_GATE_BLOCK -- gate groups per load batch in the reverse/ascending passes.
#include <cuda_runtime.h>

#include <type_traits>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "gf_common.cuh"
#include "gf_fused.cuh"
#include "gf_internal.h"

#ifndef GF_FUSED_GH
#define GF_FUSED_GH 1
#endif
#ifndef GF_FUSED_BLOCK
#define GF_FUSED_BLOCK 1  // 2: registers 100-124, 5% slower
#endif
#ifndef GF_GATE_BLOCK
#define GF_GATE_BLOCK 4
#endif
#ifndef GF_HOLE_ILP
#define GF_HOLE_ILP 2  // independent DMMA accumulator chains per hole in the split hole phase
#endif
#ifndef GF_SPARSE_DMMA_DEFAULT
#define GF_SPARSE_DMMA_DEFAULT 1  // measured: c3 -11%, c4 -11%, c5 -11% per summand vs the FMA form
#endif

// GF_CHECKS (libgfcuda_checked.so, the bounds-checked build the GPU tests run
// in place of compute-sanitizer, which this pool does not allow): device
// asserts that trap on the first violated tile / global address invariant.
#ifdef GF_CHECKS
#include <cstdio>
#define GF_DCHECK(c)                                                                        \
    do {                                                                                    \
        if (!(c)) {                                                                         \
            printf("GF_CHECKS %s:%d block (%d,%d) thread %d: %s\n", __FILE__, __LINE__,     \
                   blockIdx.x, blockIdx.y, threadIdx.x, #c);                                \
            __trap();                                                                       \
        }                                                                                   \
    } while (0)
#else
#define GF_DCHECK(c) \
    do {             \
    } while (0)
#endif

namespace gf {

// OP_REV_H: the reverse sweep of an HVP-only evaluation (no gradient hole)
enum { OP_FWD = 0, OP_FWD_DOT = 1, OP_REV_G = 2, OP_REV_GH = 3, OP_ASC_H = 4, OP_REV_H = 5 };
enum { MODE_DENSE = 0, MODE_SPARSE = 1, MODE_C1Q = 2 };

struct SweepParams {
    double2 *psi, *bra, *aux;  // [nvec][N]
    const double2 *phi0;       // [nvec][N]
    const double *weights;     // [nvec] or null
    const int64_t *basis;      // [nvec] (init kernel)
    u64 N;                     // amplitudes per vector
    u64 nunits;                // tuples (2q) or pairs (c1q) per vector
    int lo, hi;                // bit positions (c1q: lo = pa)
    int sector;
    Mat4 A, B, C;
    double *partD, *partH, *partV;  // [nvec][gridDim.x][32|32|2]
};

constexpr int kThreads = 256;

// ---------------------------------------------------------------------------
// Sweep kernel.  Grid: (ctas_per_vector, nvec).  Each CTA only touches the
// vector blockIdx.y, so every per-summand partial is independent of the batch
// composition (deterministic for any batch size / GPU count).
// ---------------------------------------------------------------------------
template <int OP, int MODE, bool FIRST>
__global__ void __launch_bounds__(kThreads) k_sweep(const SweepParams p)
{
    constexpr bool C1Q = (MODE == MODE_C1Q);
    constexpr bool SP = (MODE == MODE_SPARSE);
    constexpr int W = C1Q ? 2 : 4;  // amplitudes per unit
    constexpr bool HAS_D = (OP == OP_REV_G || OP == OP_REV_GH);
    constexpr bool HAS_H = (OP == OP_REV_GH || OP == OP_ASC_H);
    constexpr bool HAS_V = (OP == OP_FWD_DOT) || ((OP == OP_REV_G || OP == OP_REV_GH) && FIRST);

    const u64 vb = (u64)blockIdx.y * p.N;
    double2 *psi = p.psi + vb;
    double2 *bra = p.bra + vb;
    double2 *aux = p.aux + vb;
    const double2 *phi0 = p.phi0 ? p.phi0 + vb : nullptr;
    const double w = p.weights ? p.weights[blockIdx.y] : 1.0;

    double accD[32], accH[32];
    double vre = 0.0, vim = 0.0;
    if (HAS_D) {
#pragma unroll
        for (int i = 0; i < 32; ++i) accD[i] = 0.0;
    }
    if (HAS_H) {
#pragma unroll
        for (int i = 0; i < 32; ++i) accH[i] = 0.0;
    }

    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < p.nunits; t += stride) {
        u64 idx[W];
        int P = 0;
        if constexpr (C1Q) {
            u64 y0 = ins0(t, p.lo);
            idx[0] = y0;
            idx[1] = y0 | (1ull << p.lo);
            P = (__popcll(y0) & 1) ^ p.sector;
        } else {
            u64 b = ins0(ins0(t, p.lo), p.hi);
            u64 ol = 1ull << p.lo, oh = 1ull << p.hi;
            idx[0] = b;
            idx[1] = b + ol;
            idx[2] = b + oh;
            idx[3] = b + ol + oh;
        }
        double2 x[W], y[W];
#pragma unroll
        for (int i = 0; i < W; ++i) x[i] = psi[idx[i]];

        if constexpr (OP == OP_FWD || OP == OP_FWD_DOT) {
            if constexpr (C1Q) mv2(p.A, P, x, y); else mv4<SP>(p.A, x, y);
#pragma unroll
            for (int i = 0; i < W; ++i) psi[idx[i]] = y[i];
            if (OP == OP_FWD_DOT) {
#pragma unroll
                for (int i = 0; i < W; ++i) {
                    double2 f = cscale(phi0[idx[i]], w);
                    vre = fma(f.x, y[i].x, vre);
                    vre = fma(-f.y, y[i].y, vre);
                    vim = fma(f.x, y[i].y, vim);
                    vim = fma(f.y, y[i].x, vim);
                }
            }
        } else if constexpr (OP == OP_REV_G || OP == OP_REV_GH) {
            // A = G^dag (uncompute psi), B = G^T (propagate bra), C = Z^T
            double2 b[W], c[W];
#pragma unroll
            for (int i = 0; i < W; ++i) {
                if (FIRST) {
                    b[i] = cscale(phi0[idx[i]], w);
                } else {
                    b[i] = bra[idx[i]];
                }
            }
            if (HAS_V) {
#pragma unroll
                for (int i = 0; i < W; ++i) {
                    vre = fma(b[i].x, x[i].x, vre);
                    vre = fma(-b[i].y, x[i].y, vre);
                    vim = fma(b[i].x, x[i].y, vim);
                    vim = fma(b[i].y, x[i].x, vim);
                }
            }
            if constexpr (C1Q) mv2(p.A, P, x, y); else mv4<SP>(p.A, x, y);  // y = psi_l
            if constexpr (C1Q) hole_acc2(accD, P, b, y); else hole_acc(accD, b, y);
            if constexpr (OP == OP_REV_GH) {
                if (!FIRST) {
#pragma unroll
                    for (int i = 0; i < W; ++i) c[i] = aux[idx[i]];
                    if constexpr (C1Q) hole_acc2(accH, P, c, y); else hole_acc(accH, c, y);
                }
                double2 cn[W];
                if (FIRST) {
                    if constexpr (C1Q) mv2(p.C, P, b, cn); else mv4<SP>(p.C, b, cn);
                } else {
                    if constexpr (C1Q) mv2(p.B, P, c, cn); else mv4<SP>(p.B, c, cn);
                    if constexpr (C1Q) mv2_acc(p.C, P, b, cn); else mv4_acc<SP>(p.C, b, cn);
                }
#pragma unroll
                for (int i = 0; i < W; ++i) aux[idx[i]] = cn[i];
            }
            double2 bn[W];
            if constexpr (C1Q) mv2(p.B, P, b, bn); else mv4<SP>(p.B, b, bn);
#pragma unroll
            for (int i = 0; i < W; ++i) {
                psi[idx[i]] = y[i];
                bra[idx[i]] = bn[i];
            }
        } else if constexpr (OP == OP_ASC_H) {
            // A = conj(G) (recover bra), B = G (propagate v, psi), C = Z
            double2 b[W], bn[W], v[W], vn[W];
#pragma unroll
            for (int i = 0; i < W; ++i) b[i] = bra[idx[i]];
            if constexpr (C1Q) mv2(p.A, P, b, bn); else mv4<SP>(p.A, b, bn);
            if (FIRST) {
                if constexpr (C1Q) mv2(p.C, P, x, vn); else mv4<SP>(p.C, x, vn);
            } else {
#pragma unroll
                for (int i = 0; i < W; ++i) v[i] = aux[idx[i]];
                if constexpr (C1Q) hole_acc2(accH, P, bn, v); else hole_acc(accH, bn, v);
                if constexpr (C1Q) mv2(p.B, P, v, vn); else mv4<SP>(p.B, v, vn);
                if constexpr (C1Q) mv2_acc(p.C, P, x, vn); else mv4_acc<SP>(p.C, x, vn);
            }
            if constexpr (C1Q) mv2(p.B, P, x, y); else mv4<SP>(p.B, x, y);
#pragma unroll
            for (int i = 0; i < W; ++i) {
                psi[idx[i]] = y[i];
                bra[idx[i]] = bn[i];
                aux[idx[i]] = vn[i];
            }
        }
    }

    __shared__ double red[kThreads / 32 * 32];
    const u64 part = ((u64)blockIdx.y * gridDim.x + blockIdx.x);
    if (HAS_D) {
        double v = block_reduce32(accD, red);
        if (threadIdx.x < 32) p.partD[part * 32 + threadIdx.x] = v;
    }
    if (HAS_H) {
        double v = block_reduce32(accH, red);
        if (threadIdx.x < 32) p.partH[part * 32 + threadIdx.x] = v;
    }
    if (HAS_V) {
        double acc[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = 0.0;
        acc[0] = vre;
        acc[1] = vim;
        // reuse the same deterministic block reduction (entries 0,1 used)
        double v = block_reduce32(acc, red);
        if (threadIdx.x < 2) p.partV[part * 2 + threadIdx.x] = v;
    }
}


// ---------------------------------------------------------------------------
// Fused tile pass (see gf_fused.cuh).  Grid: (ctas, nvec); each CTA walks the
// tiles blockIdx.x, blockIdx.x + ctas, ... of vector blockIdx.y.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b)
{
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned ins0u(unsigned t, int b)
{
    unsigned low = t & ((1u << b) - 1u);
    return ((t >> b) << (b + 1)) | low;
}

// XOR swizzle of the tile index (double2 granularity): l ^ f(l >> 3), f a
// GF(2)-linear map onto the 16-byte slot within the 128-byte bank row.  Bit
// i >= 3 of l moves the slot by v_i = {7,5,2,7,4,6,4,3,6}[i-3], chosen by
// tools/swizzle_search.py so that the quarter-warp of a gate access (tuples
// t, t+1 x amplitudes {0, lo, hi, lo+hi}) and the half-warp of a hole access
// (tuples 4q..4q+3 x {0, lo}) hit distinct slots for the target pairs the
// pass planner emits (modelled excess wavefronts at c2: 28% -> 3% of ideal;
// the earlier fold (l>>3)^(l>>5)^(l>>7)^(l>>9) mapped bits 4, 6, 8, 10 alike).
__device__ __forceinline__ unsigned swz(unsigned l)
{
    const unsigned x = l >> 3;
    return l ^ ((__popc(x & 0x8Bu) & 1u) | ((__popc(x & 0x1ADu) & 1u) << 1) | ((__popc(x & 0x17Bu) & 1u) << 2));
}

// B fragment (two k-steps) of the real 8x8 form of a complex 4x4 gate for
// the transposed product Y^T = X^T G^T on 8-tuple groups: lane (g, t) holds
// amplitude t (re, im) of tuple g; k-step h feeds part h of that amplitude.
// G_real[(i,pi)][(j,pj)]: (0,0)=re (0,1)=-im (1,0)=im (1,1)=re.
__device__ __forceinline__ void gate_frag(const Mat4 &M, int g, int t, double &b0, double &b1)
{
    const double2 e = M.m[4 * (g >> 1) + t];
    const bool pi = g & 1;
    b0 = pi ? e.y : e.x;
    b1 = pi ? e.x : -e.y;
}

// y (this lane's amplitude) = sum of DMMA products over (x, fragment) pairs.
// GF_SPLIT_MV: the two k-steps into independent accumulators plus two DADDs
// (no DMMA -> DMMA dependency inside a gate application)
#ifndef GF_SPLIT_MV
#define GF_SPLIT_MV 0
#endif
__device__ __forceinline__ double2 dmma_mv(double2 x, double b0, double b1)
{
    double c0 = 0.0, c1 = 0.0;
#if GF_SPLIT_MV
    double d0 = 0.0, d1 = 0.0;
    dmma(c0, c1, x.x, b0);
    dmma(d0, d1, x.y, b1);
    return make_double2(c0 + d0, c1 + d1);
#else
    dmma(c0, c1, x.x, b0);
    dmma(c0, c1, x.y, b1);
    return make_double2(c0, c1);
#endif
}

__device__ __forceinline__ double2 dmma_mv2(double2 x, double b0, double b1, double2 z, double e0, double e1)
{
    double c0 = 0.0, c1 = 0.0;
#if GF_SPLIT_MV
    double d0 = 0.0, d1 = 0.0;
    dmma(c0, c1, x.x, b0);
    dmma(d0, d1, z.x, e0);
    dmma(c0, c1, x.y, b1);
    dmma(d0, d1, z.y, e1);
    return make_double2(c0 + d0, c1 + d1);
#else
    dmma(c0, c1, x.x, b0);
    dmma(c0, c1, x.y, b1);
    dmma(c0, c1, z.x, e0);
    dmma(c0, c1, z.y, e1);
    return make_double2(c0, c1);
#endif
}

// The slots of one pass applied to a tile staged in shared memory (t0 = psi,
// t1 = bra, t2 + d*T = chi_d (REV) / v_d (ASC) for ND directions); hole
// partials go to partD / partH[slot][vector][cta][32] (hole 0 = gradient D,
// hole 1 + d = HVP direction d).
template <int V>
using IC = std::integral_constant<int, V>;

template <int OP, int NT, int ND, int VAR>
__device__ __forceinline__ void run_slots(const FusedParams &p, double2 *t0, double2 *t1, double2 *t2, double *scratch,
                                          const u64 pofs, const bool accum, const int tpop, const unsigned T)
{
    constexpr int NW = NT / 32;
    constexpr int NWB = NW >= 16 ? 4 : (NW >= 8 ? 3 : (NW >= 4 ? 2 : (NW >= 2 ? 1 : 0)));  // log2(NW)
    constexpr bool HD = (OP == OP_REV_G || OP == OP_REV_GH);
    constexpr bool HH = (OP == OP_REV_GH || OP == OP_REV_H || OP == OP_ASC_H);
    constexpr bool REV = (OP == OP_REV_G || OP == OP_REV_GH || OP == OP_REV_H);
    constexpr bool CHI = (OP == OP_REV_GH || OP == OP_REV_H);  // reverse sweep carrying chi_d
    // fused gate + hole phase (dense slots): ascending sweep 3% faster; the
    // reverse sweep measured 0.5% slower with it and keeps the split phases
    constexpr bool GH = GF_FUSED_GH && (OP == OP_ASC_H);
    // VAR bit 0: the pass has parity-sparse FMA slots; bit 1: it has
    // parity-controlled one-qubit slots on the DMMA path (PM_C1QD).  Passes
    // without them compile without those branches.
    constexpr bool SPX = (VAR & 1) != 0;
    constexpr bool C1D = (VAR & 2) != 0;
    constexpr int NH = 1 + ND;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, tq = lane & 3;
    // hole operand rows: component g = 2*amp + part (re/im of one amplitude adjacent)
    const int gi = g >> 1, gpart = g & 1;
    for (int si = 0; si < p.nslots; ++si) {
        const int mode = p.ps[si].mode;
        const int zmask = p.ps[si].zmask, amask = p.ps[si].amask;
        const Mat4 &MA = p.mat[si][0];
        const Mat4 &MB = p.mat[si][1];
        const bool c1q = (mode == PM_C1Q);
        // PM_C1QD: the sector's parity-controlled 2x2 gate on local bit llo as
        // a dense 4x4 on (virtual bit lhi, llo): tuples pair two amplitude
        // pairs of opposite parity, the even-parity pair first (the sh bit of
        // odd-parity tuples is flipped), and the slot matrices are
        // V(M) = diag(M[{0,3}], M[{1,2}]) (plan side, upload_frags)
        const bool c1d = C1D && (mode == PM_C1QD);
        const unsigned nunit = c1q ? (T >> 1) : (T >> 2);
        // units per active warp: multiple of 4 (hole MMA K) -- and of 8 for the
        // 2q tensor path (8-tuple groups, paired hole MMAs)
        const unsigned TW = max(nunit / (unsigned)NW, c1q ? 4u : 8u);
        const unsigned nwa = nunit >> (31 - __clz(TW));  // powers of two
#ifdef GF_CHECKS
        {
            // every tile address below is an XOR of these columns: all < T
            // keeps every shared-memory access inside the tile
            const int ub = 31 - __clz(nunit);  // unit-index bits
            for (int i = 0; i < ub; ++i) GF_DCHECK(p.ps[si].col[i] < T);
            GF_DCHECK(p.ps[si].so < T && p.ps[si].sh < T);
            GF_DCHECK(p.ps[si].slot >= 0 && (p.ps[si].fa >= 0) && (p.ps[si].fb >= 0));
        }
#endif
        double cD0 = 0.0, cD1 = 0.0, cH0[ND], cH1[ND];
#pragma unroll
        for (int d = 0; d < ND; ++d) cH0[d] = cH1[d] = 0.0;
        if ((unsigned)warp < nwa) {
            const unsigned wbase = warp * TW;
            // GF(2)-linear unit addressing from the planner's columns:
            // A(x) = XOR of col[i] over the bits of the unit index x (tuple for
            // 2q slots, pair for c1q slots), split as A(wbase) ^ A(lane) ^ A(32k)
            const PassSlot &PS = p.ps[si];
            const int twb = 31 - __clz(TW);
            unsigned Fw = 0;
#pragma unroll
            for (int i = 0; i < NWB; ++i)
                if ((warp >> i) & 1) Fw ^= PS.col[twb + i];
            auto Alane = [&]() {
                unsigned a = 0;
#pragma unroll
                for (int i = 0; i < 5; ++i)
                    if ((lane >> i) & 1) a ^= PS.col[i];
                return a;
            };
            auto Ahi = [&](unsigned k) {  // A(32 k)
                unsigned a = 0;
#pragma unroll
                for (int i = 0; i < FMAXM - 6; ++i)
                    if ((k >> i) & 1u) a ^= PS.col[5 + i];
                return a;
            };
            if (c1q) {
                // ---- parity-controlled 1q slot (sector implicit qubit): FMA on pairs
                // (the parity of the pair index equals that of its low member:
                // inserting a zero bit keeps the popcount)
                double2 *V = (OP == OP_ASC_H) ? t1 : t0;
                const unsigned Fl = Fw ^ Alane();
                for (unsigned j = lane; j < TW; j += 32) {
                    const int P = (tpop + __popc(wbase + j)) & 1 ^ p.sector;
                    const unsigned s0 = Fl ^ Ahi(j >> 5), s1 = s0 ^ PS.so;
                    double2 x[2] = {V[s0], V[s1]}, y[2];
                    mv2(MA, P, x, y);
                    V[s0] = y[0];
                    V[s1] = y[1];
                }
                if constexpr (HD || HH) {
                    __syncwarp();
                    const double *d0 = reinterpret_cast<const double *>(t0);
                    const double *d1 = reinterpret_cast<const double *>(t1);
                    const double *d2 = reinterpret_cast<const double *>(t2);
                    const unsigned Ft = Fw ^ ((tq & 1) ? PS.col[0] : 0u) ^ ((tq & 2) ? PS.col[1] : 0u);
                    for (unsigned q = 0; q < TW / 4; ++q) {
                        unsigned s0 = Ft;
#pragma unroll
                        for (int i = 0; i < FMAXM - 3; ++i)
                            if ((q >> i) & 1u) s0 ^= PS.col[2 + i];
                        const int P = (tpop + __popc(wbase + 4 * q + tq)) & 1 ^ p.sector;
                        const int i0 = P ? 1 : 0, i1 = P ? 2 : 3;
                        const bool on = (gi == i0) || (gi == i1);
                        const int o = on ? 2 * (int)((gi == i0) ? s0 : (s0 ^ PS.so)) + gpart : 0;
                        const int li = on ? 0 : -1;
                        if constexpr (REV) {
                            const double k = li >= 0 ? d0[o] : 0.0;
                            if constexpr (HD) dmma(cD0, cD1, li >= 0 ? d1[o] : 0.0, k);
                            if constexpr (HH) {
#pragma unroll
                                for (int d = 0; d < ND; ++d)
                                    if ((amask >> d) & 1) dmma(cH0[d], cH1[d], li >= 0 ? d2[2 * d * T + o] : 0.0, k);
                            }
                        } else {
                            const double bq = li >= 0 ? d1[o] : 0.0;
#pragma unroll
                            for (int d = 0; d < ND; ++d)
                                if ((amask >> d) & 1) dmma(cH0[d], cH1[d], bq, li >= 0 ? d2[2 * d * T + o] : 0.0);
                        }
                    }
                    __syncwarp();
                }
                if constexpr (OP != OP_FWD && OP != OP_FWD_DOT) {
                    const unsigned Fl = Fw ^ Alane();
                    for (unsigned j = lane; j < TW; j += 32) {
                        const unsigned l0 = Fl ^ Ahi(j >> 5), l1 = l0 ^ PS.so;
                        const int P = (tpop + __popc(wbase + j)) & 1 ^ p.sector;
                        if constexpr (REV) {
                            double2 b[2] = {t1[l0], t1[l1]}, bn[2];
                            if constexpr (CHI) {
#pragma unroll
                                for (int d = 0; d < ND; ++d) {
                                    const bool act = (amask >> d) & 1, zz = (zmask >> d) & 1;
                                    if (!act && !zz) continue;  // chi_d stays exactly zero
                                    double2 *X = t2 + d * T;
                                    double2 cc[2] = {X[l0], X[l1]}, cn[2] = {czero(), czero()};
                                    if (act) mv2(MB, P, cc, cn);
                                    if (zz) mv2_acc(p.mat[si][2 + d], P, b, cn);
                                    X[l0] = cn[0];
                                    X[l1] = cn[1];
                                }
                            }
                            mv2(MB, P, b, bn);
                            t1[l0] = bn[0];
                            t1[l1] = bn[1];
                        } else {
                            double2 x[2] = {t0[l0], t0[l1]}, y[2];
#pragma unroll
                            for (int d = 0; d < ND; ++d) {
                                const bool act = (amask >> d) & 1, zz = (zmask >> d) & 1;
                                if (!act && !zz) continue;  // v_d stays exactly zero
                                double2 *X = t2 + d * T;
                                double2 v[2] = {X[l0], X[l1]}, vn[2] = {czero(), czero()};
                                if (act) mv2(MB, P, v, vn);
                                if (zz) mv2_acc(p.mat[si][2 + d], P, x, vn);
                                X[l0] = vn[0];
                                X[l1] = vn[1];
                            }
                            mv2(MB, P, x, y);
                            t0[l0] = y[0];
                            t0[l1] = y[1];
                        }
                    }
                }
            } else {
                // ---- two-qubit slot, all FP64 math on the tensor cores (DMMA m8n8k4).
                // Tuple -> swizzled tile index is GF(2)-linear (bit insertion +
                // XOR swizzle), so every address is an XOR of precomputed columns.
                // F(x) = swz(ins0u(ins0u(x, llo), lhi)) is GF(2)-linear in the
                // tuple index x: F(wbase | t) = F(wbase) ^ F(t) for t < TW
                const unsigned c0 = PS.col[0], c1 = PS.col[1], c2 = PS.col[2];
                const unsigned offA = ((tq & 2) ? PS.sh : 0u) ^ ((tq & 1) ? PS.so : 0u);
                // C1QD parity flips: tuple index x = warp * TW + 8 grp + g (gate /
                // update layout) or warp * TW + 4 q + tq (hole layout); a tuple's
                // even-parity pair is its low one, so odd tuples XOR sh
                const unsigned wpar = c1d ? (unsigned)((tpop + __popc((unsigned)warp) + p.sector) & 1) : 0u;
                const unsigned gparA = wpar ^ ((unsigned)__popc((unsigned)g) & 1u);
                auto flipA = [&](unsigned grp) -> unsigned {  // address XOR of group grp (gate layout)
                    if constexpr (!C1D) return 0u;
                    return (c1d && ((gparA ^ (unsigned)__popc(grp)) & 1u)) ? PS.sh : 0u;
                };
                // gate layout: lane (g, tq) = amp tq of tuple g
                const unsigned baseA = Fw ^ ((g & 1) ? c0 : 0u) ^ ((g & 2) ? c1 : 0u) ^ ((g & 4) ? c2 : 0u) ^ offA;
                const unsigned ngrp = TW >> 3;                // groups of 8 tuples
                unsigned colA[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) colA[i] = PS.col[3 + i];
                auto addrA = [&](unsigned grp) {
                    unsigned a = baseA;
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if ((grp >> i) & 1u) a ^= colA[i];
                    return a;
                };
                // offsets of group u of a block of 8 (u known at compile time in
                // the unrolled loops: one or two XORs per address, no predicates)
                auto gcomb = [&](unsigned u) {
                    return ((u & 1u) ? colA[0] : 0u) ^ ((u & 2u) ? colA[1] : 0u) ^ ((u & 4u) ? colA[2] : 0u);
                };
                double2 *V = (OP == OP_ASC_H) ? t1 : t0;
                // SPX: the pass has sparse slots; dense-only passes compile
                // without the sparse branch (it costs them registers and
                // scheduling freedom even when never taken)
                const bool sparse = SPX && (mode == PM_SPARSE);
                // this lane's DMMA B fragments, issued before the gate phase so
                // the update phase does not wait on them
                double2 fB = make_double2(0.0, 0.0), fZ[ND];
#pragma unroll
                for (int d = 0; d < ND; ++d) fZ[d] = make_double2(0.0, 0.0);
                if (!sparse) {
                    if constexpr (OP != OP_FWD && OP != OP_FWD_DOT) fB = __ldg(&p.frag[PS.fb * 32 + lane]);
                    if constexpr (CHI || OP == OP_ASC_H) {
#pragma unroll
                        for (int d = 0; d < ND; ++d) fZ[d] = __ldg(&p.frag[(PS.fz + d) * 32 + lane]);
                    }
                }
                if (sparse) {
                    // parity-conserving gates: half of G is structural zeros, so the
                    // sparse FMA form does half the flops of the dense DMMA form
                    const unsigned Fl = Fw ^ Alane();
                    for (unsigned j = lane; j < TW; j += 32) {
                        const unsigned b0 = Fl ^ Ahi(j >> 5);
                        const unsigned L[4] = {b0, b0 ^ PS.so, b0 ^ PS.sh, b0 ^ PS.so ^ PS.sh};
                        double2 x[4], y[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) x[i] = V[L[i]];
                        mv4<true>(MA, x, y);
#pragma unroll
                        for (int i = 0; i < 4; ++i) V[L[i]] = y[i];
                    }
                } else if (GH && !c1d) {
                    // ---- fused gate + holes.  The gate is C = G X with X's
                    // components as K: lane (g, tq) loads part tq&1 of amps
                    // (tq>>1) and (tq>>1)+2 of tuple g, and receives component g
                    // (amp g>>1, part g&1) of tuples 2tq and 2tq+1 -- exactly the
                    // hole MMA operand layout (tuples as K).  The new psi (reverse)
                    // / bra (ascending) feeds the hole MMAs from registers instead
                    // of being re-read from shared memory after a warp sync.
                    const double2 fA2 = __ldg(&p.frag[PS.fa2 * 32 + lane]);
                    const unsigned inB = Fw ^ ((g & 1) ? c0 : 0u) ^ ((g & 2) ? c1 : 0u) ^ ((g & 4) ? c2 : 0u) ^
                                         ((tq & 2) ? PS.so : 0u);
                    const unsigned outA = Fw ^ ((tq & 1) ? c1 : 0u) ^ ((tq & 2) ? c2 : 0u) ^ ((g & 2) ? PS.so : 0u) ^
                                          ((g & 4) ? PS.sh : 0u);
                    const int ipart = tq & 1, opart = g & 1;
                    double *Vd = reinterpret_cast<double *>(V);
                    double eD0 = 0.0, eD1 = 0.0, eH0[ND], eH1[ND];  // tuples 2tq+1 (ILP)
#pragma unroll
                    for (int d = 0; d < ND; ++d) eH0[d] = eH1[d] = 0.0;
                    // GF_FUSED_BLOCK groups at a time: all shared-memory loads first
                    // (the compiler cannot prove the groups disjoint from the
                    // stores), then the gate MMAs, the stores, the hole MMAs
                    auto fused_loop = [&](auto AC) {
                        constexpr int A = decltype(AC)::value;
                        constexpr unsigned FB = GF_FUSED_BLOCK;
                        const double *hd = reinterpret_cast<const double *>(REV ? t1 : t2);
                        for (unsigned gb = 0; gb < ngrp; gb += FB) {
                            double x0[FB], x1[FB], ha0[FB], ha1[FB], hb0[ND][FB], hb1[ND][FB];
                            unsigned o0[FB], o1[FB];
#pragma unroll
                            for (unsigned u = 0; u < FB; ++u) {
                                if (gb + u >= ngrp) continue;  // tiny tiles
                                const unsigned go = addrA(gb + u) ^ baseA;
                                const unsigned ei = inB ^ go, eo = outA ^ go;
                                o0[u] = 2 * eo + opart;
                                o1[u] = 2 * (eo ^ c0) + opart;
                                x0[u] = Vd[2 * ei + ipart];
                                x1[u] = Vd[2 * (ei ^ PS.sh) + ipart];
                                if constexpr (REV && HD) {
                                    ha0[u] = hd[o0[u]];
                                    ha1[u] = hd[o1[u]];
                                }
#pragma unroll
                                for (int d = 0; d < ND; ++d) {
                                    if (!HH || !(A == 2 ? ((amask >> d) & 1) : A)) continue;
                                    const double *cd = reinterpret_cast<const double *>(t2 + d * T);
                                    hb0[d][u] = cd[o0[u]];
                                    hb1[d][u] = cd[o1[u]];
                                }
                            }
#pragma unroll
                            for (unsigned u = 0; u < FB; ++u) {
                                if (gb + u >= ngrp) continue;
                                double y0 = 0.0, y1 = 0.0;
                                dmma(y0, y1, fA2.x, x0[u]);
                                dmma(y0, y1, fA2.y, x1[u]);
                                Vd[o0[u]] = y0;
                                Vd[o1[u]] = y1;
                                if constexpr (REV) {
                                    if constexpr (HD) {
                                        dmma(cD0, cD1, ha0[u], y0);
                                        dmma(eD0, eD1, ha1[u], y1);
                                    }
                                    if constexpr (HH) {
#pragma unroll
                                        for (int d = 0; d < ND; ++d) {
                                            if (!(A == 2 ? ((amask >> d) & 1) : A)) continue;
                                            dmma(cH0[d], cH1[d], hb0[d][u], y0);
                                            dmma(eH0[d], eH1[d], hb1[d][u], y1);
                                        }
                                    }
                                } else {
#pragma unroll
                                    for (int d = 0; d < ND; ++d) {
                                        if (!(A == 2 ? ((amask >> d) & 1) : A)) continue;
                                        dmma(cH0[d], cH1[d], y0, hb0[d][u]);
                                        dmma(eH0[d], eH1[d], y1, hb1[d][u]);
                                    }
                                }
                            }
                        }
                        (void)hd;
                    };
                    if constexpr (ND == 1 && HH) {
                        if (amask & 1) fused_loop(IC<1>{});
                        else fused_loop(IC<0>{});
                    } else {
                        fused_loop(IC<2>{});
                    }
                    cD0 += eD0;
                    cD1 += eD1;
#pragma unroll
                    for (int d = 0; d < ND; ++d) {
                        cH0[d] += eH0[d];
                        cH1[d] += eH1[d];
                    }
                } else {
                    // coalesced per-lane fragment rows (a dynamically indexed
                    // Mat4 in parameter space serialises 16 ways in the
                    // constant cache)
                    const double2 fA = __ldg(&p.frag[p.ps[si].fa * 32 + lane]);
                    const double fa0 = fA.x, fa1 = fA.y;
                    if constexpr (OP == OP_FWD || OP == OP_FWD_DOT) {
                        // forward passes: register-bound occupancy, one group at a time
                        for (unsigned gb = 0; gb < ngrp; gb += 8) {
                            const unsigned ab = addrA(gb);
#pragma unroll
                            for (unsigned u = 0; u < 8; ++u) {
                                if (gb + u >= ngrp) break;  // ngrp < 8 only for tiny tiles
                                const unsigned ad = ab ^ gcomb(u) ^ flipA(gb + u);
                                V[ad] = dmma_mv(V[ad], fa0, fa1);
                            }
                        }
                    } else {
                        // loads of a block of groups first, then the MMAs and
                        // stores: the groups are disjoint, but the compiler cannot
                        // prove it and otherwise serialises load -> MMA -> store
                        // per group (reverse sweep 1.6% faster at 4; 8 and the
                        // same blocking of the update phase raise the registers
                        // to the 128 cap and run slower)
                        constexpr unsigned GB = GF_GATE_BLOCK;
                        for (unsigned gb = 0; gb < ngrp; gb += GB) {
                            const unsigned ab = addrA(gb & ~7u) ^ gcomb(gb & 7u);
                            const unsigned nb = min(GB, ngrp - gb);  // < GB only for tiny tiles
                            double2 xv[GB];
#pragma unroll
                            for (unsigned u = 0; u < GB; ++u)
                                if (u < nb) xv[u] = V[ab ^ gcomb(u) ^ flipA(gb + u)];
#pragma unroll
                            for (unsigned u = 0; u < GB; ++u)
                                if (u < nb) V[ab ^ gcomb(u) ^ flipA(gb + u)] = dmma_mv(xv[u], fa0, fa1);
                        }
                    }
                }
                if constexpr (HD || HH) if (!GH || sparse || c1d) {
                    __syncwarp();
                    // hole layout: lane (g, tq) = component g (amp g>>1, part g&1) of tuple tq
                    const unsigned offH = ((gi & 2) ? PS.sh : 0u) ^ ((gi & 1) ? PS.so : 0u);
                    const unsigned baseH = Fw ^ ((tq & 1) ? c0 : 0u) ^ ((tq & 2) ? c1 : 0u) ^ offH;
                    unsigned colH[5];
#pragma unroll
                    for (int i = 0; i < 5; ++i) colH[i] = PS.col[2 + i];
                    const double *d0 = reinterpret_cast<const double *>(t0) + gpart;
                    const double *d1 = reinterpret_cast<const double *>(t1) + gpart;
                    const double *d2 = reinterpret_cast<const double *>(t2) + gpart;
                    double eD0 = 0.0, eD1 = 0.0, eH0[ND], eH1[ND];  // second accumulators (ILP)
#pragma unroll
                    for (int d = 0; d < ND; ++d) eH0[d] = eH1[d] = 0.0;
#if GF_HOLE_ILP >= 4
                    // third / fourth accumulator sets for u & 2 (independent DMMA chains)
                    double fD0 = 0.0, fD1 = 0.0, gD0 = 0.0, gD1 = 0.0, fH0[ND], fH1[ND], gH0[ND], gH1[ND];
#pragma unroll
                    for (int d = 0; d < ND; ++d) fH0[d] = fH1[d] = gH0[d] = gH1[d] = 0.0;
#endif
                    const unsigned nq = TW >> 2;
                    // C1QD: parity of tuple 4q + tq is hpar ^ popc(q); a1 = tuple q + 1 (q even)
                    const unsigned hpar = wpar ^ ((unsigned)__popc((unsigned)tq) & 1u);
                    auto flipH = [&](unsigned q) -> unsigned {
                        if constexpr (!C1D) return 0u;
                        return (c1d && ((hpar ^ (unsigned)__popc(q)) & 1u)) ? PS.sh : 0u;
                    };
                    // AC: 1/0 = direction active/inactive known at compile time
                    // (ND == 1, hoisted out of the loop), 2 = test amask per d
                    auto hole_loop = [&](auto AC) {
                        constexpr int A = decltype(AC)::value;
                        for (unsigned qb = 0; qb < nq; qb += 8) {
                          unsigned ab = baseH;
#pragma unroll
                          for (int i = 3; i < 5; ++i)
                              if ((qb >> i) & 1u) ab ^= colH[i];
#pragma unroll
                          for (unsigned u = 0; u < 8; u += 2) {
                            const unsigned q = qb + u;
                            if (q >= nq) break;  // nq < 8 only for tiny tiles
                            const unsigned a0 = ab ^ ((u & 2u) ? colH[1] : 0u) ^ ((u & 4u) ? colH[2] : 0u) ^ flipH(q);
                            const unsigned a1 = a0 ^ colH[0] ^ flipH(q) ^ flipH(q + 1);
                            const unsigned o0 = 2 * a0, o1 = 2 * a1;
#if GF_HOLE_ILP >= 4
                            const bool alt = (u & 2u) != 0;  // compile-time in the unrolled loop
                            double &xD0 = alt ? fD0 : cD0, &xD1 = alt ? fD1 : cD1;
                            double &yD0 = alt ? gD0 : eD0, &yD1 = alt ? gD1 : eD1;
                            double *xH0 = alt ? fH0 : cH0, *xH1 = alt ? fH1 : cH1;
                            double *yH0 = alt ? gH0 : eH0, *yH1 = alt ? gH1 : eH1;
#else
                            double &xD0 = cD0, &xD1 = cD1, &yD0 = eD0, &yD1 = eD1;
                            double *xH0 = cH0, *xH1 = cH1, *yH0 = eH0, *yH1 = eH1;
#endif
                            if constexpr (REV) {
                                const double k0 = d0[o0], k1 = d0[o1];
                                if constexpr (HD) {
                                    dmma(xD0, xD1, d1[o0], k0);
                                    dmma(yD0, yD1, d1[o1], k1);
                                }
                                if constexpr (HH) {
#pragma unroll
                                    for (int d = 0; d < ND; ++d) {
                                        if (!(A == 2 ? ((amask >> d) & 1) : A)) continue;
                                        dmma(xH0[d], xH1[d], d2[2 * d * T + o0], k0);
                                        dmma(yH0[d], yH1[d], d2[2 * d * T + o1], k1);
                                    }
                                }
                            } else {
                                const double b0 = d1[o0], b1 = d1[o1];
#pragma unroll
                                for (int d = 0; d < ND; ++d) {
                                    if (!(A == 2 ? ((amask >> d) & 1) : A)) continue;
                                    dmma(xH0[d], xH1[d], b0, d2[2 * d * T + o0]);
                                    dmma(yH0[d], yH1[d], b1, d2[2 * d * T + o1]);
                                }
                            }
                          }
                        }
                    };
                    if constexpr (ND == 1 && HH) {
                        if (amask & 1) hole_loop(IC<1>{});
                        else hole_loop(IC<0>{});
                    } else {
                        hole_loop(IC<2>{});
                    }
#if GF_HOLE_ILP >= 4
                    cD0 += fD0;
                    cD1 += fD1;
                    eD0 += gD0;
                    eD1 += gD1;
#pragma unroll
                    for (int d = 0; d < ND; ++d) {
                        cH0[d] += fH0[d];
                        cH1[d] += fH1[d];
                        eH0[d] += gH0[d];
                        eH1[d] += gH1[d];
                    }
#endif
                    cD0 += eD0;
                    cD1 += eD1;
#pragma unroll
                    for (int d = 0; d < ND; ++d) {
                        cH0[d] += eH0[d];
                        cH1[d] += eH1[d];
                    }
                    __syncwarp();
                }
                if constexpr (GH) if (!sparse && !c1d) __syncwarp();  // fused phase reads precede the updates' writes
                if constexpr (OP != OP_FWD && OP != OP_FWD_DOT) if (sparse) {
                    const unsigned Fl = Fw ^ Alane();
                    for (unsigned j = lane; j < TW; j += 32) {
                        const unsigned b0 = Fl ^ Ahi(j >> 5);
                        const unsigned L[4] = {b0, b0 ^ PS.so, b0 ^ PS.sh, b0 ^ PS.so ^ PS.sh};
                        if constexpr (REV) {
                            double2 bb[4], bn[4];
#pragma unroll
                            for (int i = 0; i < 4; ++i) bb[i] = t1[L[i]];
                            if constexpr (CHI) {
#pragma unroll
                                for (int d = 0; d < ND; ++d) {
                                    const bool act = (amask >> d) & 1, zz = (zmask >> d) & 1;
                                    if (!act && !zz) continue;
                                    double2 *X = t2 + d * T;
                                    double2 cc[4], cn[4];
#pragma unroll
                                    for (int i = 0; i < 4; ++i) {
                                        cc[i] = X[L[i]];
                                        cn[i] = czero();
                                    }
                                    if (act) mv4<true>(MB, cc, cn);
                                    if (zz) mv4_acc<true>(p.mat[si][2 + d], bb, cn);
#pragma unroll
                                    for (int i = 0; i < 4; ++i) X[L[i]] = cn[i];
                                }
                            }
                            mv4<true>(MB, bb, bn);
#pragma unroll
                            for (int i = 0; i < 4; ++i) t1[L[i]] = bn[i];
                        } else {
                            double2 x[4], y[4];
#pragma unroll
                            for (int i = 0; i < 4; ++i) x[i] = t0[L[i]];
#pragma unroll
                            for (int d = 0; d < ND; ++d) {
                                const bool act = (amask >> d) & 1, zz = (zmask >> d) & 1;
                                if (!act && !zz) continue;
                                double2 *X = t2 + d * T;
                                double2 v[4], vn[4];
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    v[i] = X[L[i]];
                                    vn[i] = czero();
                                }
                                if (act) mv4<true>(MB, v, vn);
                                if (zz) mv4_acc<true>(p.mat[si][2 + d], x, vn);
#pragma unroll
                                for (int i = 0; i < 4; ++i) X[L[i]] = vn[i];
                            }
                            mv4<true>(MB, x, y);
#pragma unroll
                            for (int i = 0; i < 4; ++i) t0[L[i]] = y[i];
                        }
                    }
                } else {
                    double fc0[ND], fc1[ND];
                    const double fb0 = fB.x, fb1 = fB.y;
#pragma unroll
                    for (int d = 0; d < ND; ++d) {
                        fc0[d] = fZ[d].x;
                        fc1[d] = fZ[d].y;
                    }
                    // AC / ZC: 1/0 = chi_d (v_d) active / Z_d nonzero known at
                    // compile time (ND == 1, hoisted), 2 = test the masks per d
                    auto grp_loop = [&](auto AC, auto ZC) {
                        constexpr int A = decltype(AC)::value, Z = decltype(ZC)::value;
                        for (unsigned gb = 0; gb < ngrp; gb += 8) {
                          const unsigned ab = addrA(gb);
#pragma unroll
                          for (unsigned u = 0; u < 8; ++u) {
                            if (gb + u >= ngrp) break;  // ngrp < 8 only for tiny tiles
                            const unsigned ad = ab ^ gcomb(u) ^ flipA(gb + u);
                            const double2 x = REV ? t1[ad] : t0[ad];
                            if constexpr (CHI || OP == OP_ASC_H) {
#pragma unroll
                                for (int d = 0; d < ND; ++d) {
                                    const bool act = A == 2 ? ((amask >> d) & 1) : A;
                                    const bool zz = Z == 2 ? ((zmask >> d) & 1) : Z;
                                    double2 *X = t2 + d * T;
                                    if (act && zz) X[ad] = dmma_mv2(X[ad], fb0, fb1, x, fc0[d], fc1[d]);
                                    else if (act) X[ad] = dmma_mv(X[ad], fb0, fb1);
                                    else if (zz) X[ad] = dmma_mv(x, fc0[d], fc1[d]);
                                }
                            }
                            if constexpr (REV) t1[ad] = dmma_mv(x, fb0, fb1);
                            else t0[ad] = dmma_mv(x, fb0, fb1);
                          }
                        }
                    };
                    // Paired parity blocks (sector / parity circuits, one direction):
                    // G and Z are block diagonal over amplitude pairs E, O, and
                    // both act on the same input x (bra / psi), so one DMMA per
                    // block with B = [M1_b | M2_b] yields x' and the Z term, and a
                    // second with B = [0 | M1_b] adds M1 X: 4 DMMAs per group for
                    // x' and X' instead of 6.  Lane (g, t) feeds component t&1 of
                    // amplitude b[t>>1] and receives x' (t < 2) or X' (t >= 2) of
                    // amplitude b[t&1].
                    auto pair_loop = [&](auto AC, auto ZC) {
                        constexpr int A = decltype(AC)::value, Z = decltype(ZC)::value;
                        const double2 fE = __ldg(&p.frag[PS.fpe * 32 + lane]);
                        const double2 fO = __ldg(&p.frag[(PS.fpe + 1) * 32 + lane]);
                        auto offamp = [&](int a) -> unsigned {
                            return ((a & 2) ? PS.sh : 0u) ^ ((a & 1) ? PS.so : 0u);
                        };
                        // block amplitudes: parity {0,3} / {1,2}; C1QD virtual {0,1} / {2,3}
                        const int eIn = PS.pblk ? (tq >> 1) : ((tq >> 1) ? 3 : 0);
                        const int oIn = PS.pblk ? 2 + (tq >> 1) : ((tq >> 1) ? 2 : 1);
                        const int eOut = PS.pblk ? (tq & 1) : ((tq & 1) ? 3 : 0);
                        const int oOut = PS.pblk ? 2 + (tq & 1) : ((tq & 1) ? 2 : 1);
                        const unsigned dEi = offamp(eIn) ^ offA, dOi = offamp(oIn) ^ offA;
                        const unsigned dEo = offamp(eOut) ^ offA, dOo = offamp(oOut) ^ offA;
                        const int part = tq & 1;
                        double2 *xt = REV ? t1 : t0;
                        double2 *Xt = t2;
                        const double *xd = reinterpret_cast<const double *>(xt);
                        const double *Xd = reinterpret_cast<const double *>(Xt);
                        double2 *dE = (tq < 2) ? xt : Xt;
                        const bool storeX = (tq < 2) || A || Z;
                        for (unsigned gb = 0; gb < ngrp; gb += 8) {
                          const unsigned ab = addrA(gb);
#pragma unroll
                          for (unsigned u = 0; u < 8; ++u) {
                            if (gb + u >= ngrp) break;
                            const unsigned ad = ab ^ gcomb(u) ^ flipA(gb + u);  // lane's own amplitude
                            const double xe = xd[2 * (ad ^ dEi) + part], xo = xd[2 * (ad ^ dOi) + part];
                            double Xe = 0.0, Xo = 0.0;
                            if (A) {
                                Xe = Xd[2 * (ad ^ dEi) + part];
                                Xo = Xd[2 * (ad ^ dOi) + part];
                            }
                            double e0 = 0.0, e1 = 0.0, o0 = 0.0, o1 = 0.0;
                            dmma(e0, e1, xe, fE.x);
                            dmma(o0, o1, xo, fO.x);
                            if (A) {
                                dmma(e0, e1, Xe, fE.y);
                                dmma(o0, o1, Xo, fO.y);
                            }
                            if (storeX) {
                                dE[ad ^ dEo] = make_double2(e0, e1);
                                dE[ad ^ dOo] = make_double2(o0, o1);
                            }
                          }
                        }
                    };
                    if constexpr (C1D && ND == 1 && (CHI || OP == OP_ASC_H)) {
                        if (PS.pair) {
                            const bool a = amask & 1, z = zmask & 1;
                            if (a) pair_loop(IC<1>{}, IC<1>{});  // Z = 0 rows are zero in the fragment
                            else if (z) pair_loop(IC<0>{}, IC<1>{});
                            else pair_loop(IC<0>{}, IC<0>{});
                        }
                    }
                    if (C1D && ND == 1 && (CHI || OP == OP_ASC_H) && PS.pair) {
                        // done above
                    } else if constexpr (ND == 1 && (CHI || OP == OP_ASC_H)) {
                        const bool a = amask & 1, z = zmask & 1;
                        if (a && z) grp_loop(IC<1>{}, IC<1>{});
                        else if (a) grp_loop(IC<1>{}, IC<0>{});
                        else if (z) grp_loop(IC<0>{}, IC<1>{});
                        else grp_loop(IC<0>{}, IC<0>{});
                    } else {
                        grp_loop(IC<2>{}, IC<2>{});
                    }
                }
            }
        }
        if constexpr (HD || HH) {
            // Fold the 8x8 real fragment to the complex 4x4 hole inside the warp:
            // lane (2i, j) holds C[2i][2j..2j+1], its partner lane (2i+1, j)
            // C[2i+1][2j..2j+1]; Re D_ij = C[2i][2j] - C[2i+1][2j+1],
            // Im D_ij = C[2i][2j+1] + C[2i+1][2j].  The even-g lanes store 32
            // doubles per warp and hole into the slot-parity half of scratch,
            // so one barrier per slot orders both the tile and the partials:
            // scratch[s & 1] is next written at slot s + 2, after the barrier of
            // slot s + 1, which the reducing warps pass only after reducing.
            double *sbuf = scratch + (si & 1) * (NH * NW * 32);
            // C1QD slots: virtual entry (i', j') is full-space entry (m(i'), m(j')),
            // m = [0, 3, 1, 2]; cross-block entries (different environments) are
            // the exactly-zero off-pattern entries of the full-space hole
            const bool c1dh = C1D && (mode == PM_C1QD);
            auto fold_store = [&](int hole, double c0, double c1) {
                const double o0 = __shfl_xor_sync(0xffffffffu, c0, 4);
                const double o1 = __shfl_xor_sync(0xffffffffu, c1, 4);
                if (!(g & 1)) {
                    const int iv = g >> 1, jv = tq;
                    int e = iv * 4 + jv;
                    bool keep = true;
                    if (c1dh) {
                        const int mi = (0x2130 >> (4 * iv)) & 3, mj = (0x2130 >> (4 * jv)) & 3;  // m = [0,3,1,2]
                        e = mi * 4 + mj;
                        keep = (iv >> 1) == (jv >> 1);
                    }
                    double *dst = sbuf + (hole * NW + warp) * 32 + e * 2;
                    dst[0] = keep ? c0 - o1 : 0.0;
                    dst[1] = keep ? c1 + o0 : 0.0;
                }
            };
            if ((unsigned)warp < nwa) {
                if (HD) fold_store(0, cD0, cD1);
                if (HH) {
#pragma unroll
                    for (int d = 0; d < ND; ++d) fold_store(1 + d, cH0[d], cH1[d]);
                }
            }
            __syncthreads();
            if (tid < 32 * NH) {
                const int hole = tid >> 5;
                if ((hole == 0 && HD) || (hole >= 1 && HH)) {
                    const int i = tid & 31;
                    double sum = 0.0;
                    for (unsigned ww = 0; ww < nwa; ++ww) sum += sbuf[(hole * NW + ww) * 32 + i];
                    // this CTA's partial of this slot (accumulated over its tiles in
                    // tile order; one tile per CTA by default)
                    double *dst = (hole == 0 ? p.partD : p.partH + (u64)(hole - 1) * p.hstride) +
                                  (u64)p.ps[si].slot * p.nvec * p.ctas * 32 + pofs + i;
                    *dst = accum ? *dst + sum : sum;
                }
            }
        } else {
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// Parity-structured passes on the FP64 FMA pipe (PM_UNIT slots, VAR == 4).
//
// A parity-conserving 4x4 gate is two 2x2 blocks (amplitudes {0,3} and {1,2});
// in a parity sector the gates on the implicit qubit are 2x2 blocks selected
// by the pair's parity.  Both are *units*: two amplitudes a0, a1 = a0 ^ so and
// a block selector b that picks the 2x2 block of every slot matrix and the
// 2x2 sub-block of the 4x4 hole.  An m8n8k4 DMMA cannot skip the zero blocks
// (it executes twice the algorithmic flops, and B200's DMMA and DFMA share
// one FP64 datapath), so these passes use FMAs: a lane owns units with a fixed
// b (lane bit 0; its 2x2 blocks live in registers for the whole slot), loads
// the unit's amplitudes of psi / bra / chi once, does the gate, the hole
// accumulations and the updates in registers, and stores them once -- 96 DFMA
// and 12 conflict-free 128-bit shared accesses per unit of a reverse slot,
// against 12 DMMAs (= 192 DFMA-equivalents) and 18 wavefronts on the dense
// path.  B = conj(A) in both sweeps (G^T = conj(G^dag), G = conj(conj G)), so
// only A and Z are held.
// ---------------------------------------------------------------------------
#ifndef GF_UNIT_WIDTH
#define GF_UNIT_WIDTH 2  // 128-thread variant: units per step (independent chains), as many again loading
#endif

// c + conj(a) * b
__device__ __forceinline__ double2 cfmac(double2 a, double2 b, double2 c)
{
    c.x = fma(a.x, b.x, c.x);
    c.x = fma(a.y, b.y, c.x);
    c.y = fma(a.x, b.y, c.y);
    c.y = fma(-a.y, b.x, c.y);
    return c;
}
// conj(a) * b
__device__ __forceinline__ double2 cmulc(double2 a, double2 b)
{
    return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.x, b.y, -a.y * b.x));
}

// First-unit tile index of every (slot, thread) of a unit pass: unit index =
// [warp >> 1][unit of the lane][lane][b = warp & 1], address = XOR of the
// slot's columns over its set bits (tile-invariant; shared memory table).
template <int NT>
__device__ __forceinline__ void unit_bases(const FusedParams &p, unsigned short *ubase, const unsigned T)
{
    constexpr int NW = NT / 32;
    const unsigned nunit = T >> 1;
    const unsigned TW = max(nunit / (unsigned)NW, 32u);
    const int itb = 31 - __clz(TW >> 5);
    for (int e = threadIdx.x; e < p.nslots * NT; e += NT) {
        const int si = e / NT, t = e % NT, lane = t & 31, warp = t >> 5;
        const PassSlot &PS = p.ps[si];
        unsigned a = (warp & 1) ? PS.col[0] : 0u;
        for (int i = 0; i < 5; ++i)
            if ((lane >> i) & 1) a ^= PS.col[1 + i];
        for (int i = 0; i < 3; ++i)
            if ((warp >> (1 + i)) & 1) a ^= PS.col[min(6 + itb + i, FMAXM - 2)];
        ubase[e] = (unsigned short)a;
    }
}

template <int OP, int NT>
__device__ __forceinline__ void run_units(const FusedParams &p, double2 *t0, double2 *t1, double2 *t2, double *scratch,
                                          const unsigned short *ubase, const u64 pofs, const bool accum,
                                          const int tpop, const unsigned T)
{
    constexpr int NW = NT / 32;
    constexpr bool FWD = (OP == OP_FWD || OP == OP_FWD_DOT);
    constexpr bool HD = (OP == OP_REV_G || OP == OP_REV_GH);
    constexpr bool HH = (OP == OP_REV_GH || OP == OP_REV_H || OP == OP_ASC_H);
    constexpr bool REV = (OP == OP_REV_G || OP == OP_REV_GH || OP == OP_REV_H);
    constexpr bool CHI = (OP == OP_REV_GH || OP == OP_REV_H);
    constexpr bool ASC = (OP == OP_ASC_H);
    constexpr int NH = 2;
    // units per step: 128-thread CTAs (two warps per scheduler) work on two
    // units at a time with the next two loading; wider CTAs on one with the
    // next one loading
    constexpr int W = (NT <= 128) ? GF_UNIT_WIDTH : 1;
    const int tid = threadIdx.x, lane = tid & 31;
    // warp-uniform warp index: the block selector b = warp & 1 is uniform, so
    // the 2x2 blocks of the slot matrices are uniform-register FMA operands
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
    const int b = warp & 1;
    const unsigned nunit = T >> 1;
    const unsigned TW = max(nunit / (unsigned)NW, 32u);  // units per active warp
    const unsigned nwa = nunit >> (31 - __clz(TW));      // >= 2 (tiles of >= 2^7 amplitudes)
    const unsigned nit = TW >> 5;  // units per lane: a power of two, <= 8 for every tile shape
    const int itb = 31 - __clz(nit);
    const unsigned tpar = (unsigned)((tpop ^ p.sector) & 1);
    struct Unit {
        double2 x0, x1, b0, b1, c0, c1;
        unsigned a0, a1;
    };
    for (int si = 0; si < p.nslots; ++si) {
        const PassSlot &PS = p.ps[si];
#ifdef GF_CHECKS
        {
            const int ub = 31 - __clz(nunit);
            for (int i = 0; i < ub; ++i) GF_DCHECK(PS.col[i] < T);
            GF_DCHECK(PS.so < T && PS.so != 0u && PS.mode == PM_UNIT && nit <= 8u && nwa >= 2u);
        }
#endif
        // this CTA's running partial of the slot (tiles after its first): read
        // early, added after the barrier
        double prev = 0.0;
        double *pdst = nullptr;
        if constexpr (HD || HH) {
            if (tid < 32 * NH) {
                const int hole = tid >> 5;
                if ((hole == 0 && HD) || (hole >= 1 && HH)) {
                    pdst = (hole == 0 ? p.partD : p.partH) + (u64)PS.slot * p.nvec * p.ctas * 32 + pofs + (tid & 31);
                    if (accum) prev = *pdst;
                }
            }
        }
        double2 dD[W][4], dH[W][4];
#pragma unroll
        for (int k = 0; k < W; ++k)
#pragma unroll
            for (int i = 0; i < 4; ++i) dD[k][i] = dH[k][i] = czero();
        if ((unsigned)warp < nwa) {
            // block b of A = mat[0] and Z = mat[2]: rows / columns {0, 3} or {1, 2}
            const int i0 = b ? 1 : 0, i1 = b ? 2 : 3;
            const Mat4 &MA = p.mat[si][0];
            const double2 a00 = MA.m[4 * i0 + i0], a01 = MA.m[4 * i0 + i1];
            const double2 a10 = MA.m[4 * i1 + i0], a11 = MA.m[4 * i1 + i1];
            double2 z00 = czero(), z01 = czero(), z10 = czero(), z11 = czero();
            if constexpr (CHI || ASC) {
                const Mat4 &MZ = p.mat[si][2];
                z00 = MZ.m[4 * i0 + i0]; z01 = MZ.m[4 * i0 + i1];
                z10 = MZ.m[4 * i1 + i0]; z11 = MZ.m[4 * i1 + i1];
            }
            const unsigned dso = PS.so;
            // unit index = [warp >> 1][unit of the lane][lane][b]
            // (tabulated once per CTA by unit_bases; parity-controlled slots
            // add the tile's parity)
            unsigned a = (unsigned)ubase[si * NT + tid] ^ ((PS.upar && tpar) ? PS.col[0] : 0u);
            // the lane's units in Gray-code order: one XOR per unit
            const unsigned g0 = PS.col[6], g1 = PS.col[7], g2 = PS.col[8];
            unsigned cnt = 0;
            auto advance = [&]() {
                ++cnt;
                a ^= (cnt & 1u) ? g0 : ((cnt & 2u) ? g1 : g2);
            };
            auto load = [&](Unit &u) {
                u.a0 = a;
                u.a1 = a ^ dso;
                GF_DCHECK(u.a0 < T && u.a1 < T);
                u.x0 = t0[u.a0];
                u.x1 = t0[u.a1];
                if constexpr (!FWD) {
                    u.b0 = t1[u.a0];
                    u.b1 = t1[u.a1];
                }
                if constexpr (CHI || ASC) {
                    u.c0 = t2[u.a0];
                    u.c1 = t2[u.a1];
                }
                advance();
            };
            auto work = [&](const Unit &u, double2 *eD, double2 *eH) {
                if constexpr (FWD) {
                    t0[u.a0] = cfma(a01, u.x1, cmul(a00, u.x0));
                    t0[u.a1] = cfma(a11, u.x1, cmul(a10, u.x0));
                } else if constexpr (REV) {
                    // psi <- G^dag psi
                    const double2 y0 = cfma(a01, u.x1, cmul(a00, u.x0));
                    const double2 y1 = cfma(a11, u.x1, cmul(a10, u.x0));
                    t0[u.a0] = y0;
                    t0[u.a1] = y1;
                    if constexpr (HD) {  // D += hole(bra, psi)
                        eD[0] = cfma(u.b0, y0, eD[0]);
                        eD[1] = cfma(u.b0, y1, eD[1]);
                        eD[2] = cfma(u.b1, y0, eD[2]);
                        eD[3] = cfma(u.b1, y1, eD[3]);
                    }
                    if constexpr (CHI) {  // H += hole(chi, psi); chi <- G^T chi + Z^T bra
                        eH[0] = cfma(u.c0, y0, eH[0]);
                        eH[1] = cfma(u.c0, y1, eH[1]);
                        eH[2] = cfma(u.c1, y0, eH[2]);
                        eH[3] = cfma(u.c1, y1, eH[3]);
                        double2 n0 = cfma(z01, u.b1, cmul(z00, u.b0));
                        double2 n1 = cfma(z11, u.b1, cmul(z10, u.b0));
                        n0 = cfmac(a01, u.c1, cfmac(a00, u.c0, n0));
                        n1 = cfmac(a11, u.c1, cfmac(a10, u.c0, n1));
                        t2[u.a0] = n0;
                        t2[u.a1] = n1;
                    }
                    // bra <- G^T bra
                    t1[u.a0] = cfmac(a01, u.b1, cmulc(a00, u.b0));
                    t1[u.a1] = cfmac(a11, u.b1, cmulc(a10, u.b0));
                } else {
                    // bra <- conj(G) bra; H += hole(bra, v); v <- G v + Z psi; psi <- G psi
                    const double2 q0 = cfma(a01, u.b1, cmul(a00, u.b0));
                    const double2 q1 = cfma(a11, u.b1, cmul(a10, u.b0));
                    t1[u.a0] = q0;
                    t1[u.a1] = q1;
                    eH[0] = cfma(q0, u.c0, eH[0]);
                    eH[1] = cfma(q0, u.c1, eH[1]);
                    eH[2] = cfma(q1, u.c0, eH[2]);
                    eH[3] = cfma(q1, u.c1, eH[3]);
                    double2 n0 = cfma(z01, u.x1, cmul(z00, u.x0));
                    double2 n1 = cfma(z11, u.x1, cmul(z10, u.x0));
                    n0 = cfmac(a01, u.c1, cfmac(a00, u.c0, n0));
                    n1 = cfmac(a11, u.c1, cfmac(a10, u.c0, n1));
                    t2[u.a0] = n0;
                    t2[u.a1] = n1;
                    t0[u.a0] = cfmac(a01, u.x1, cmulc(a00, u.x0));
                    t0[u.a1] = cfmac(a11, u.x1, cmulc(a10, u.x0));
                }
            };
            if (nit >= 2u * W) {
                // W units per step (independent FMA chains and accumulator
                // sets), the next W already loading
                Unit u[2][W];
#pragma unroll
                for (int k = 0; k < W; ++k) load(u[0][k]);
                for (unsigned it = 0; it < nit; it += 2 * W) {
#pragma unroll
                    for (int k = 0; k < W; ++k) load(u[1][k]);
#pragma unroll
                    for (int k = 0; k < W; ++k) work(u[0][k], dD[k], dH[k]);
                    if (it + 2 * W < nit) {
#pragma unroll
                        for (int k = 0; k < W; ++k) load(u[0][k]);
                    }
#pragma unroll
                    for (int k = 0; k < W; ++k) work(u[1][k], dD[k], dH[k]);
                }
            } else {
                for (unsigned it = 0; it < nit; ++it) {
                    Unit u;
                    load(u);
                    work(u, dD[0], dH[0]);
                }
            }
            if constexpr (W > 1) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    dD[0][i] = cadd(dD[0][i], dD[W - 1][i]);
                    dH[0][i] = cadd(dH[0][i], dH[W - 1][i]);
                }
            }
        }
        if constexpr (HD || HH) {
            // Per hole a lane holds the 2x2 complex block of the warp's b as 8
            // doubles v[4 r + 2 s + part].  Reduce-scatter over lane bits 4 (r),
            // 3 (s), 2 (part), then add over bits 1 and 0 (fixed order:
            // deterministic); lanes (b4 b3 b2 0 0) write entry (r, s, part) to
            // scratch[hole][warp][8].  Entry (r, s) of block b is entry
            // (i_r, i_s) of the 4x4 hole, (i_0, i_1) = b ? (1, 2) : (0, 3).
            double *sbuf = scratch + (si & 1) * (NH * NW * 8);
            auto fold_store = [&](int hole, const double2 d[4]) {
                double v[8] = {d[0].x, d[0].y, d[1].x, d[1].y, d[2].x, d[2].y, d[3].x, d[3].y};
#pragma unroll
                for (int s = 16, half = 4; s >= 4; s >>= 1, half >>= 1) {
                    const bool upper = (lane & s) != 0;
#pragma unroll
                    for (int i = 0; i < half; ++i) {
                        const double send = upper ? v[i] : v[i + half];
                        const double keep = upper ? v[i + half] : v[i];
                        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
                    }
                }
                double tot = v[0] + __shfl_xor_sync(0xffffffffu, v[0], 2);
                tot += __shfl_xor_sync(0xffffffffu, tot, 1);
                if (!(lane & 3)) sbuf[(hole * NW + warp) * 8 + (lane >> 2)] = tot;
            };
            if ((unsigned)warp < nwa) {
                if constexpr (HD) fold_store(0, dD[0]);
                if constexpr (HH) fold_store(1, dH[0]);
            }
            __syncthreads();
            if (pdst) {
                const int hole = tid >> 5, i = tid & 31;
                const int row = i >> 3, colm = (i >> 1) & 3, part = i & 1;
                const int rb = (row == 1 || row == 2), cb = (colm == 1 || colm == 2);
                double sum = 0.0;
                if (rb == cb) {  // on-pattern entry of block rb
                    const int q = 4 * (row >> 1) + 2 * (colm >> 1) + part;  // r = (row >= 2), s = (col >= 2)
                    for (unsigned ww = rb; ww < nwa; ww += 2) sum += sbuf[(hole * NW + ww) * 8 + q];
                }
                *pdst = prev + sum;
            }
        } else {
            __syncthreads();
        }
    }
}

// (measured: asking for 4 CTAs per SM in the forward passes, <= 64 registers,
// left the forward sweep unchanged -- 24.1 vs 23.6 TFLOP/s)
// GF_NT512_M11 (experiment): 512-thread CTAs at two per SM for the 2^11-tile
// passes -- 32 warps per SM instead of 16, at <= 64 registers per thread
#ifndef GF_NT512_M11
#define GF_NT512_M11 0
#endif
// (unit passes: the forward sweep holds one vector per tile and is bound by
// HBM / shared-memory traffic -- GF_UNIT_FWD_CTAS CTAs of 256 threads per SM)
#ifndef GF_UNIT_FWD_CTAS
#define GF_UNIT_FWD_CTAS 4
#endif
template <int OP, bool FIRST, int NT, int ND, int VAR>
__global__ void __launch_bounds__(NT, (GF_NT512_M11 && NT == 512) ? 2
                                      : ((VAR == 4 && NT < 256) ? 2
                                         : ((VAR == 4 && NT == 256 && OP <= OP_FWD_DOT) ? GF_UNIT_FWD_CTAS : 512 / NT)))
    k_fused(const FusedParams p)
{
    constexpr int NW = NT / 32;  // warps per CTA
    constexpr int NH = 1 + ND;   // hole slots: gradient + ND directions
    constexpr int NV = (OP == OP_FWD || OP == OP_FWD_DOT) ? 1 : (OP == OP_REV_G ? 2 : 2 + ND);
    constexpr bool HD = (OP == OP_REV_G || OP == OP_REV_GH || OP == OP_REV_H);  // value on the first reverse pass
        constexpr bool HV = (OP == OP_FWD_DOT) || (HD && FIRST);
    constexpr bool REV = (OP == OP_REV_G || OP == OP_REV_GH || OP == OP_REV_H);
    extern __shared__ __align__(16) unsigned char fsm[];
    const int m = p.m, c = p.c;
    const unsigned T = 1u << m;
    double2 *t0 = reinterpret_cast<double2 *>(fsm);  // psi
    double2 *t1 = t0 + T;                            // bra
    double2 *t2 = t0 + 2 * T;                        // chi_d (REV) / v_d (ASC), ND tiles
    double *scratch = reinterpret_cast<double *>(t0 + NV * T);  // [NH][NW][64]; unit passes [2][NH][NW][8]
    u64 *hiofs = reinterpret_cast<u64 *>(scratch + (VAR == 4 ? 2 * NH * NW * 8 : NH * NW * 64));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // A CTA whose tiles are all dead (light cone, below) has nothing to do
    // outside a sweep's first pass: leave before building the tables.  Its
    // hole partials are exact zeros.
    if constexpr (!FIRST) {
        if (p.fixmask) {
            const u64 jb0 = (u64)p.basis[blockIdx.y];
            bool any = false;
            for (u64 tile = blockIdx.x; tile < p.ntiles && !any; tile += gridDim.x) {
                u64 base = 0;
                for (int i = 0; i < p.nglob; ++i)
                    if ((tile >> i) & 1ull) base |= 1ull << p.gpos[i];
                any = ((jb0 ^ base) & p.fixmask) == 0ull;
            }
            if (!any) {
                constexpr bool HDP = (OP == OP_REV_G || OP == OP_REV_GH);
                constexpr bool HHP = (OP == OP_REV_GH || OP == OP_REV_H || OP == OP_ASC_H);
                if constexpr (HDP || HHP) {
                    const u64 pofs = ((u64)blockIdx.y * p.ctas + blockIdx.x) * 32;
                    for (int e = tid; e < p.nslots * 32 * NH; e += NT) {
                        const int si = e / (32 * NH), hole = (e / 32) % NH, i = e & 31;
                        if ((hole == 0 && HDP) || (hole >= 1 && HHP)) {
                            double *dst = (hole == 0 ? p.partD : p.partH + (u64)(hole - 1) * p.hstride) +
                                          (u64)p.ps[si].slot * p.nvec * p.ctas * 32 + pofs + i;
                            *dst = 0.0;
                        }
                    }
                }
                if constexpr (HV) {
                    if (tid < 2) p.partV[((u64)blockIdx.y * p.ctas + blockIdx.x) * 2 + tid] = 0.0;
                }
                return;
            }
        }
    }
    // unit passes: per-(slot, thread) tile index of the thread's first unit
    unsigned short *ubase = reinterpret_cast<unsigned short *>(hiofs + (1 << (p.m - p.c)));
    if constexpr (VAR == 4) unit_bases<NT>(p, ubase, T);
    const u64 vb = (u64)blockIdx.y * p.N;
    double2 *psi = p.psi + vb;
    double2 *bra = p.bra + vb;
    double2 *aux = p.aux + vb;
    const double2 *phi0 = p.phi0 ? p.phi0 + vb : nullptr;
    const double w = p.weights ? p.weights[blockIdx.y] : 1.0;

    const int nh = 1 << (m - c);
    for (int h = tid; h < nh; h += NT) {
        u64 o = 0;
        for (int i = 0; i < m - c; ++i)
            if ((h >> i) & 1) o |= 1ull << p.lpos[c + i];
        hiofs[h] = o;
    }
    __syncthreads();
    double vre = 0.0, vim = 0.0;
    const unsigned cmask = (1u << c) - 1u;
    // swz is GF(2)-linear and l = tid ^ (l - tid) in the tile loops below
    const unsigned stid = swz((unsigned)tid);
    auto sw = [&](unsigned l) { return stid ^ swz(l ^ (unsigned)tid); };

    // the first forward and first ascending passes start from psi_0 = |j>
    constexpr bool SYNTH = (OP == OP_FWD || OP == OP_FWD_DOT || OP == OP_ASC_H) && FIRST;
    constexpr bool FWDOP = (OP == OP_FWD || OP == OP_FWD_DOT);
    constexpr bool ASC = (OP == OP_ASC_H);
    const u64 jb = (u64)p.basis[blockIdx.y];
    auto tile_base = [&](u64 tile) {
        u64 base = 0;
        for (int i = 0; i < p.nglob; ++i)
            if ((tile >> i) & 1ull) base |= 1ull << p.gpos[i];
        return base;
    };
    // Light cone of the basis state (p.fixmask, plan_passes).  The forward
    // states psi (and the forward tangent v) of summand j vanish wherever a
    // qubit b that no applied slot has touched differs from j.  A tile whose
    // global bits disagree with j on such a qubit is *dead*:
    //  * psi = v = 0 on it before and after the pass, so its holes are zero;
    //  * no remaining slot of the sweep touches b, so nothing ever flows from
    //    the tile's amplitudes into amplitudes that agree with j on b: chi on
    //    them is never read against a nonzero psi;
    //  * the reverse pass and the ascending pass that replays it have the same
    //    tiles and fixmask, and on one tile they are exact inverses on the bra
    //    (conj(G) G^T = 1), with everything in between nested inside them:
    //    skipping both leaves the bra of every later pass unchanged.
    // So a dead tile is skipped altogether -- no loads, no slots, no stores --
    // except in the first pass of a sweep, which initialises HBM: zeros for
    // psi (forward, ascending) and chi / v, w phi0 for the bra.
    auto is_live = [&](u64 base) { return ((jb ^ base) & p.fixmask) == 0ull; };
    const int sm = p.store_mask;
    // Element l of a live tile: plain copies go global -> shared with cp.async
    // (no register round trip, every element in flight at once); the
    // synthesised |j> and the zero chi / v are written by the thread.
    auto load_elem = [&](u64 a, unsigned sl, bool live) {
        GF_DCHECK(a < p.N && sl < T);
        if constexpr (SYNTH)
            t0[sl] = make_double2(a == jb ? 1.0 : 0.0, 0.0);  // psi_0 = |j>, no HBM read
        else if (live)
            cp_async16(&t0[sl], &psi[a]);
        if constexpr (NV >= 2) {
            if constexpr (!(REV && FIRST)) {
                if (live) cp_async16(&t1[sl], &bra[a]);
            } else {
                if (!p.weights) cp_async16(&t1[sl], &phi0[a]);  // bra_0 = phi0 (unit weight): plain copy
            }
        }
        if constexpr (NV >= 3) {
#pragma unroll
            for (int d = 0; d < ND; ++d) {
                if constexpr (FIRST) t2[d * T + sl] = czero();
                else if (live) cp_async16(&t2[d * T + sl], &aux[a + d * p.auxstride]);
            }
        }
    };
    if (p.exp_noio) {
        for (unsigned l = tid; l < NV * T; l += NT) t0[l] = czero();
    } else if (blockIdx.x < p.ntiles) {
        const u64 base = tile_base(blockIdx.x);
        const bool live = is_live(base);
        if (live || FIRST)
            for (unsigned l = tid; l < T; l += NT) load_elem(base + (l & cmask) + hiofs[l >> c], sw(l), live);
    }
    cp_async_commit();

    for (u64 tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
        const u64 base = tile_base(tile);
        const int tpop = __popcll(tile);
        const bool live = is_live(base);
        if constexpr (REV && FIRST) {
            // bra_0 = w phi0; the value <phi0|psi_n> is read back from the tile
            if (p.weights) {
                for (unsigned l = tid; l < T; l += NT) {
                    const u64 a = base + (l & cmask) + hiofs[l >> c];
                    t1[sw(l)] = cscale(phi0[a], w);
                }
            }
            cp_async_wait<0>();
            for (unsigned l = tid; l < T && live; l += NT) {
                const unsigned sl = sw(l);
                const double2 x = t0[sl], b = t1[sl];
                vre = fma(b.x, x.x, vre);
                vre = fma(-b.y, x.y, vre);
                vim = fma(b.x, x.y, vim);
                vim = fma(b.y, x.x, vim);
            }
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();

        const u64 pofs = ((u64)blockIdx.y * p.ctas + blockIdx.x) * 32;
        if (live) {
            if constexpr (VAR == 4)
                run_units<OP, NT>(p, t0, t1, t2, scratch, ubase, pofs, tile != blockIdx.x, tpop, T);
            else
                run_slots<OP, NT, ND, VAR>(p, t0, t1, t2, scratch, pofs, tile != blockIdx.x, tpop, T);
        } else if constexpr (!FWDOP) {
            // the hole partials of a dead tile are exact zeros
            if (tile == blockIdx.x) {
                constexpr bool HDP = (OP == OP_REV_G || OP == OP_REV_GH);
                constexpr bool HHP = (OP == OP_REV_GH || OP == OP_REV_H || OP == OP_ASC_H);
                for (int e = tid; e < p.nslots * 32 * NH; e += NT) {
                    const int si = e / (32 * NH), hole = (e / 32) % NH, i = e & 31;
                    if ((hole == 0 && HDP) || (hole >= 1 && HHP)) {
                        double *dst = (hole == 0 ? p.partD : p.partH + (u64)(hole - 1) * p.hstride) +
                                      (u64)p.ps[si].slot * p.nvec * p.ctas * 32 + pofs + i;
                        *dst = 0.0;
                    }
                }
            }
        }

        // Write the tile back and, element by element, start the next tile's
        // load into the slot just read: every thread reloads exactly the
        // elements it stored, so no barrier separates the two tiles (the last
        // slot's barrier ordered the tile writes before these reads; the wait +
        // barrier at the top of the next trip publishes the new tile).
        const u64 next = tile + gridDim.x;
        const bool more = next < p.ntiles && !p.exp_noio;
        const u64 nbase = more ? tile_base(next) : 0ull;
        const bool nlive = more ? is_live(nbase) : true;
        const bool reload = more && (nlive || FIRST);
        // dead tile in a first pass: zeros for psi (synthesised sweeps) and chi / v, w phi0 for the bra
        const bool wpsi = (sm & 1) && (live || SYNTH);
        const bool wbra = (sm & 2) && (live || (REV && FIRST));
        const bool waux = (sm & 4) && (live || FIRST);
        const bool skip = !live && !FIRST;  // nothing was loaded, nothing changes
        for (unsigned l = tid; l < T && !p.exp_noio; l += NT) {
            const u64 o = (l & cmask) + hiofs[l >> c];
            const u64 a = base + o;
            const unsigned sl = sw(l);
            if (!skip) {
                if (wpsi) psi[a] = t0[sl];
                if constexpr (NV >= 2) if (wbra) bra[a] = t1[sl];
                if constexpr (NV >= 3) {
                    if (waux) {
#pragma unroll
                        for (int d = 0; d < ND; ++d) aux[a + d * p.auxstride] = t2[d * T + sl];
                    }
                }
                if constexpr (OP == OP_FWD_DOT) {
                    if (live) {
                        const double2 x = t0[sl];
                        const double2 f = cscale(phi0[a], w);
                        vre = fma(f.x, x.x, vre);
                        vre = fma(-f.y, x.y, vre);
                        vim = fma(f.x, x.y, vim);
                        vim = fma(f.y, x.x, vim);
                    }
                }
            }
            if (reload) load_elem(nbase + o, sl, nlive);
        }
        if (p.exp_noio && next < p.ntiles) {
            __syncthreads();
            for (unsigned l = tid; l < NV * T; l += NT) t0[l] = czero();
        }
        cp_async_commit();
    }

    if constexpr (HV) {
        vre = warp_sum(vre);
        vim = warp_sum(vim);
        __syncthreads();
        if (lane == 0) {
            scratch[warp * 2] = vre;
            scratch[warp * 2 + 1] = vim;
        }
        __syncthreads();
        if (tid < 2) {
            double s = 0.0;
            for (int ww = 0; ww < NT / 32; ++ww) s += scratch[ww * 2 + tid];
            p.partV[((u64)blockIdx.y * p.ctas + blockIdx.x) * 2 + tid] = s;
        }
    }
    // per-CTA partials are summed in ascending CTA order by k_reduce_ctas after
    // the sweeps (a last-CTA reduction here cost every CTA a memory fence)
}


// |j> for every vector of the batch (basis index per vector).
__global__ void k_init_basis(double2 *psi, u64 N, const int64_t *basis, int64_t nvec)
{
    const u64 total = N * (u64)nvec;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (u64)gridDim.x * blockDim.x) {
        u64 b = i / N, x = i - b * N;
        psi[i] = make_double2((int64_t)x == basis[b] ? 1.0 : 0.0, 0.0);
    }
}

// part[s][b][c][32] -> q[s][b][32], summing c ascending.
// q[sb][e] = sum over c ascending of part[sb][c][e], e < ne (32 for a hole, 2 for the value)
__global__ void k_reduce_ctas(const double *part, double *q, int64_t nsb, int ctas, int ne = 32)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nsb * ne) return;
    int64_t sb = i / ne;
    int e = (int)(i - sb * ne);
    const double *src = part + sb * ctas * ne + e;
    double acc = 0.0;
    for (int c = 0; c < ctas; ++c) acc += src[(int64_t)c * ne];
    q[i] = acc;
}

// Chunk records.  rec = [value(2)] [D: nlog*32] [H: nlog*32].  One warp per
// record entry: lanes stride over the chunk's summands, then a fixed xor tree
// (deterministic, independent of batch boundaries since chunks are aligned).
__global__ void k_chunk_records(const double *qD, const double *qHd, const double *qHa, const double *partV,
                                int64_t nvec, int ctas, int nslots, int nlog, const int *lstart,
                                const int *lslots, const int *swapped, int chunk, int flags, int parity_only,
                                int nd, int64_t qhstride, double *out)
{
    const int rec = 2 + 32 * nlog * (1 + nd);
    const int64_t nchunks = (nvec + chunk - 1) / chunk;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nchunks * rec) return;
    const int64_t ch = w / rec;
    const int r = (int)(w - ch * rec);
    const int64_t b0 = ch * chunk, b1 = (nvec < b0 + chunk) ? nvec : (b0 + chunk);
    double acc = 0.0;
    if (r < 2) {
        if (partV) {
            for (int64_t b = b0 + lane; b < b1; b += 32)
                for (int c = 0; c < ctas; ++c) acc += partV[(b * ctas + c) * 2 + r];
        }
    } else {
        int rr = r - 2;
        const int blk = rr / (32 * nlog);  // 0 = gradient D, 1 + d = HVP direction d
        rr -= blk * 32 * nlog;
        const bool isH = blk >= 1;
        const int64_t hoff = isH ? (int64_t)(blk - 1) * qhstride : 0;
        const int l = rr >> 5, q = rr & 31;
        const int e = q >> 1, ri = q & 1;
        const int ii = e >> 2, jj = e & 3;
        const double *src = isH ? qHd + hoff : qD;
        // compressed-sector hole entries pairing opposite-parity rows/cols
        // would pair different implicit-qubit values: exactly zero in the
        // full-space sum (both vectors live in the sector)
        const bool offpat = parity_only && (((ii ^ (ii >> 1)) & 1) != ((jj ^ (jj >> 1)) & 1));
        const bool want = (isH ? (flags & 4) : (flags & 2)) && !offpat;
        if (want) {
            for (int64_t b = b0 + lane; b < b1; b += 32)
                for (int t = lstart[l]; t < lstart[l + 1]; ++t) {
                    int s = lslots[t];
                    int si = ii, sj = jj;
                    if (swapped[s]) {  // WIRE_SWAP = [0,2,1,3]
                        si = (ii == 1) ? 2 : (ii == 2 ? 1 : ii);
                        sj = (jj == 1) ? 2 : (jj == 2 ? 1 : jj);
                    }
                    int64_t o = ((int64_t)s * nvec + b) * 32 + 2 * (4 * si + sj) + ri;
                    acc += src[o];
                    if (isH) acc += qHa[hoff + o];
                }
        }
    }
    acc = warp_sum(acc);
    if (lane == 0) out[w] = acc;
}

// per-slot sums over the batch: q[s][b][32] -> out[s][32]
__global__ void k_slot_sums(const double *q, const double *q2, int64_t nvec, int nslots, int parity_only,
                            double *out)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nslots * 32) return;
    int s = i >> 5, e = i & 31;
    int ii = (e >> 1) >> 2, jj = (e >> 1) & 3;
    double acc = 0.0;
    if (parity_only && (((ii ^ (ii >> 1)) & 1) != ((jj ^ (jj >> 1)) & 1))) {
        out[i] = 0.0;
        return;
    }
    for (int64_t b = 0; b < nvec; ++b) {
        acc += q[((int64_t)s * nvec + b) * 32 + e];
        if (q2) acc += q2[((int64_t)s * nvec + b) * 32 + e];
    }
    out[i] = acc;
}

}  // namespace gf

using namespace gf;

// ---------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------
struct SlotInfo {
    int q1, q2;  // normalised q1 < q2 (full-space qubits)
    bool swapped;
    int logical;
    int mode_c1q;  // touches the implicit qubit in sector mode
    int lo, hi;    // bit positions in the stored (compressed) space
};

struct gf_plan {
    int k, K, sector, n, nlog, chunk;
    int64_t max_batch;
    u64 N;
    int ctas;
    std::vector<SlotInfo> slots;
    std::vector<Mat4> G, Gd, Gt, Gc, Z, Zt;  // per slot, normalised orientation (direction 0)
    std::vector<char> spG, spZ;
    bool have_z = false;
    int nd = 1;                                           // HVP directions per sweep
    std::vector<Mat4> Zm[FMAXDIR], Ztm[FMAXDIR];          // per direction, per slot
    std::vector<char> spZm[FMAXDIR], nzZm[FMAXDIR];       // parity zeros / any nonzero
    int aux_dirs = 1;                                     // directions the aux workspace holds
    double2 *psi = nullptr, *bra = nullptr, *aux = nullptr;
    double *partD = nullptr, *partHd = nullptr, *partHa = nullptr, *partV = nullptr;
    double *qD = nullptr, *qHd = nullptr, *qHa = nullptr, *qV = nullptr;
    int *d_lstart = nullptr, *d_lslots = nullptr, *d_swapped = nullptr;
    int64_t last_launches = 0;
    int last_flags = 0;
    // fused tile engine
    bool fused = false;
    bool sparse_fma = true;  // parity-sparse slots as FMA (else dense DMMA with structural zeros)
    bool c1q_dmma = true;    // parity-controlled 1q slots on the DMMA path (PM_C1QD) instead of FMA pairs
    bool pair_blocks = false; // paired parity-block DMMAs in the update phases (PassSlot::pair; GF_PAIR_BLOCKS=1)
    bool lightcone = true;    // skip the psi / v work of tiles outside the basis state's light cone (GF_LIGHTCONE)
    bool unit_fma = false;    // sector plans: every slot as FP64-FMA units (PM_UNIT, run_units) when nd == 1
    int unit_nt = 256;        // threads per CTA of the unit passes (GF_UNIT_NT)
    int fm = 0, fc = 0;
    // geometry only (matrices filled per eval).  The ascending HVP sweep must
    // replay exactly the reverse slot order of the reverse sweep (the two HVP
    // half-sums are only order-invariant together), so asc_passes is
    // rev_passes reversed with each pass's slot list reversed.
    std::vector<FusedParams> fwd_passes, rev_passes, asc_passes;
    // multi-direction sweeps (2 + nd vectors per tile) on 2^10 tiles: two CTAs
    // per SM instead of one (c2 full Hessian 120 s -> 112 s)
    std::vector<FusedParams> rev_md, asc_md;
    // per-lane DMMA B fragments of every slot matrix, [slot][FK_*][32 lanes]
    // (double2 = the two k-steps); rebuilt on the eval stream when dirty
    double2 *d_frag = nullptr;
    std::vector<double2> h_frag;
    bool frag_dirty = true;
    // optional phase timing (CUDA events on the eval stream)
    bool profiling = false;
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    double phase_ms[4] = {0, 0, 0, 0};  // accumulated: forward, reverse, ascending, reduce
    // one event set per profiled evaluation, collected without a host sync per
    // evaluation (ev / ev_rev1 alias the current set)
    struct EvSet {
        cudaEvent_t ev[5];
        cudaEvent_t rev1;
        bool has_rev1;
    };
    std::vector<EvSet> evsets;
    size_t ev_used = 0;
    // the first reverse pass alone (the sweep's dominant launch: every tile is live)
    cudaEvent_t ev_rev1 = nullptr;
    bool rev1_pending = false;
    double rev1_ms = 0.0;
    int64_t rev1_launches = 0, rev1_vectors = 0;
    int rev1_slots = 0;
    int64_t phase_launches[4] = {0, 0, 0, 0};
    int pending = 0;
};

static Mat4 to_mat4(const double *m)
{
    Mat4 r;
    for (int e = 0; e < 16; ++e) r.m[e] = make_double2(m[2 * e], m[2 * e + 1]);
    return r;
}

static Mat4 wire_swap(const Mat4 &a)
{
    static const int s[4] = {0, 2, 1, 3};
    Mat4 r;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) r.m[4 * i + j] = a.m[4 * s[i] + s[j]];
    return r;
}

static Mat4 transpose(const Mat4 &a)
{
    Mat4 r;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) r.m[4 * i + j] = a.m[4 * j + i];
    return r;
}

static Mat4 conjugate(const Mat4 &a)
{
    Mat4 r;
    for (int e = 0; e < 16; ++e) r.m[e] = make_double2(a.m[e].x, -a.m[e].y);
    return r;
}

static bool parity_zeros(const Mat4 &a)
{
    static const int off[8] = {1, 2, 4, 7, 8, 11, 13, 14};
    for (int e : off)
        if (a.m[e].x != 0.0 || a.m[e].y != 0.0) return false;
    return true;
}

#define GF_CUDA(call)                                                                   \
    do {                                                                                \
        cudaError_t _e = (call);                                                        \
        if (_e != cudaSuccess) {                                                        \
            gf_set_error("%s:%d CUDA error %s (%s)", __FILE__, __LINE__,                \
                         cudaGetErrorName(_e), cudaGetErrorString(_e));                 \
            return _e == cudaErrorMemoryAllocation ? GF_ENOMEM : GF_ECUDA;             \
        }                                                                               \
    } while (0)

// host mirror of gate_frag for every lane
static void frag_rows(const Mat4 &M, double2 *row)
{
    for (int lane = 0; lane < 32; ++lane) {
        const int g = lane >> 2, t = lane & 3;
        const double2 e = M.m[4 * (g >> 1) + t];
        const bool pi = g & 1;
        row[lane] = make_double2(pi ? e.y : e.x, pi ? e.x : -e.y);
    }
}

// the same matrix as the A operand of C = G X on 8-tuple groups: lane (g, t)
// holds row g (component g = 2 amp + part of the output) at columns t and
// t + 4 (k-steps 0 and 1) of G's real 8x8 form
static void frag_rows_A(const Mat4 &M, double2 *row)
{
    for (int lane = 0; lane < 32; ++lane) {
        const int g = lane >> 2, t = lane & 3;
        double v[2];
        for (int h = 0; h < 2; ++h) {
            const int i = g >> 1, pp = g & 1, j = (t + 4 * h) >> 1, q = t & 1;
            const double2 e = M.m[4 * i + j];
            v[h] = (pp == q) ? e.x : (pp == 0 ? -e.y : e.y);
        }
        row[lane] = make_double2(v[0], v[1]);
    }
}

// Paired parity-block B fragments (PassSlot::pair): block b (0 = E, 1 = O) of
// the amplitude pairs {0,3} / {1,2} (pblk 0) or {0,1} / {2,3} (pblk 1); lane
// (g, t) holds B[k = t][n = g] for the x input (.x: [M1_b | M2_b]) and the X
// input (.y: [0 | M1_b]), k = 2 j' + q (input amplitude j' of the block, part
// q), n = 2 i' + p for n < 4 (x' amplitude i', part p), 4 + 2 i' + p for X'.
static void frag_rows_pair(const Mat4 &M1, const Mat4 &M2, int pblk, int blk, double2 *row)
{
    const int amps[2][2][2] = {{{0, 3}, {1, 2}}, {{0, 1}, {2, 3}}};
    const int *b = amps[pblk][blk];
    auto real = [&](const Mat4 &M, int i, int p, int j, int q) {
        const double2 m = M.m[4 * b[i] + b[j]];
        return p == q ? m.x : (p == 0 ? -m.y : m.y);
    };
    for (int lane = 0; lane < 32; ++lane) {
        const int n = lane >> 2, k = lane & 3, jj = k >> 1, q = k & 1;
        const int i = (n & 3) >> 1, pp = n & 1;
        const double bx = n < 4 ? real(M1, i, pp, jj, q) : real(M2, i, pp, jj, q);
        const double by = n < 4 ? 0.0 : real(M1, i, pp, jj, q);
        row[lane] = make_double2(bx, by);
    }
}

static int upload_frags(gf_plan *p, cudaStream_t st)
{
    if (!p->frag_dirty && p->d_frag) return GF_OK;
    const int n = std::max(1, p->n);
    const size_t rows = (size_t)n * NFK;
    if (!p->d_frag) {
        cudaError_t e = cudaMalloc(&p->d_frag, rows * 32 * sizeof(double2));
        if (e != cudaSuccess) return gf_fail(GF_ENOMEM, "fragment table: %s", cudaGetErrorString(e));
    }
    p->h_frag.assign(rows * 32, make_double2(0.0, 0.0));
    // C1QD slots: V(M) = diag(M[{0,3}], M[{1,2}]) in the virtual (partner bit,
    // explicit bit) basis; V commutes with transpose / conjugation
    auto vm = [&](int s, const Mat4 &M) {
        if (!(p->c1q_dmma && p->slots[s].mode_c1q)) return M;
        static const int m[4] = {0, 3, 1, 2};
        Mat4 r;
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j)
                r.m[4 * i + j] = ((i >> 1) == (j >> 1)) ? M.m[4 * m[i] + m[j]] : make_double2(0.0, 0.0);
        return r;
    };
    auto put = [&](int s, int kind, const std::vector<Mat4> &v) {
        if ((size_t)s < v.size()) frag_rows(vm(s, v[s]), &p->h_frag[((size_t)s * NFK + kind) * 32]);
    };
    for (int s = 0; s < p->n; ++s) {
        put(s, FK_G, p->G);
        put(s, FK_GD, p->Gd);
        put(s, FK_GT, p->Gt);
        put(s, FK_GC, p->Gc);
        if ((size_t)s < p->Gd.size()) frag_rows_A(vm(s, p->Gd[s]), &p->h_frag[((size_t)s * NFK + FK_GDA) * 32]);
        if ((size_t)s < p->Gc.size()) frag_rows_A(vm(s, p->Gc[s]), &p->h_frag[((size_t)s * NFK + FK_GCA) * 32]);
        if ((size_t)s < p->G.size() && p->have_z && (size_t)s < p->Zm[0].size()) {
            const int pblk = (p->c1q_dmma && p->slots[s].mode_c1q) ? 1 : 0;
            frag_rows_pair(vm(s, p->Gt[s]), vm(s, p->Ztm[0][s]), pblk, 0, &p->h_frag[((size_t)s * NFK + FK_PRE) * 32]);
            frag_rows_pair(vm(s, p->Gt[s]), vm(s, p->Ztm[0][s]), pblk, 1, &p->h_frag[((size_t)s * NFK + FK_PRO) * 32]);
            frag_rows_pair(vm(s, p->G[s]), vm(s, p->Zm[0][s]), pblk, 0, &p->h_frag[((size_t)s * NFK + FK_PAE) * 32]);
            frag_rows_pair(vm(s, p->G[s]), vm(s, p->Zm[0][s]), pblk, 1, &p->h_frag[((size_t)s * NFK + FK_PAO) * 32]);
        }
        for (int d = 0; d < FMAXDIR; ++d) {
            put(s, FK_ZT + d, p->Ztm[d]);
            put(s, FK_Z + d, p->Zm[d]);
        }
    }
    // pageable source: the copy is staged before the call returns, so the
    // host mirror can be rebuilt at once
    cudaError_t e = cudaMemcpyAsync(p->d_frag, p->h_frag.data(), rows * 32 * sizeof(double2),
                                    cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return gf_fail(GF_ECUDA, "fragment upload: %s", cudaGetErrorString(e));
    p->frag_dirty = false;
    return GF_OK;
}

static void plan_free(gf_plan *p)
{
    cudaFree(p->d_frag);
    for (auto &es : p->evsets) {
        for (auto &e : es.ev)
            if (e) cudaEventDestroy(e);
        if (es.rev1) cudaEventDestroy(es.rev1);
    }
    p->evsets.clear();
    void *ptrs[] = {p->psi, p->bra, p->aux, p->partD, p->partHd, p->partHa, p->partV,
                    p->qD, p->qHd, p->qHa, p->qV, p->d_lstart, p->d_lslots, p->d_swapped};
    for (void *q : ptrs)
        if (q) cudaFree(q);
}

static std::vector<FusedParams> plan_passes(const gf_plan *p, bool reverse, int m, bool unit = false);

// Environment knobs of the plan (diagnostics / experiments; the defaults are
// the measured best), parsed in one place for gf_plan_create and the
// host-only gf_plan_layout query.  The Python plan cache keys on the same
// variables (objective.py _PLAN_KNOBS).
struct PlanKnobs {
    bool stream;       // GF_ENGINE=stream: one launch per slot
    int fm;            // GF_FUSED_M: tile bits of the three-vector sweeps (default 11)
    int fc;            // GF_FUSED_C: always-local low bits (default 3 = 128 B runs)
    int fwm;           // GF_FWD_M: tile bits of the forward sweep (default fm)
    long long ctas;    // GF_FUSED_CTAS: CTAs per vector (default 148 x 8)
    bool sparse_dmma;  // GF_SPARSE_DMMA: parity-sparse slots on the DMMA path
    bool c1q_dmma;     // GF_C1Q_DMMA: parity-controlled 1q slots on the DMMA path
    bool pair_blocks;  // GF_PAIR_BLOCKS: paired parity-block DMMAs in the update phases
    bool lightcone;    // GF_LIGHTCONE: dead-tile skipping (FusedParams::fixmask)
    bool sector_fma;   // GF_SECTOR_FMA: parity-sector passes as FP64-FMA units (PM_UNIT)
    int unit_nt;       // GF_UNIT_NT: threads per CTA of those passes (256, or 128)
};

static PlanKnobs plan_knobs(int K, int tile_bits)
{
    PlanKnobs k;
    const char *eng = getenv("GF_ENGINE");
    k.stream = eng && strcmp(eng, "stream") == 0;
    const char *fmenv = getenv("GF_FUSED_M");
    const int fm = tile_bits > 0 ? tile_bits : (fmenv ? atoi(fmenv) : 11);  // 2^11: three vectors, 2 CTAs/SM
    k.fm = std::max(5, std::min(std::min(fm, FMAXM), K));
    const char *fcenv = getenv("GF_FUSED_C");
    k.fc = std::min(fcenv ? std::max(1, atoi(fcenv)) : 3, k.fm);
    const char *fwenv = getenv("GF_FWD_M");
    k.fwm = (fwenv && tile_bits <= 0) ? std::max(k.fc, std::min(std::min(atoi(fwenv), FMAXM), K)) : k.fm;
    const char *cenv = getenv("GF_FUSED_CTAS");
    k.ctas = cenv ? std::max(1ll, atoll(cenv)) : 148ll * 8;  // all tiles, up to 8 per SM
    const char *sd = getenv("GF_SPARSE_DMMA");
    k.sparse_dmma = sd ? atoi(sd) != 0 : GF_SPARSE_DMMA_DEFAULT;
    const char *cq = getenv("GF_C1Q_DMMA");
    k.c1q_dmma = cq ? atoi(cq) != 0 : true;
    const char *pb = getenv("GF_PAIR_BLOCKS");
    k.pair_blocks = pb ? atoi(pb) != 0 : false;  // measured slower: c5 5.33 vs 5.01 s, c3 11.4 vs 10.6 ms
    const char *lc = getenv("GF_LIGHTCONE");
    k.lightcone = lc ? atoi(lc) != 0 : true;
    const char *sf = getenv("GF_SECTOR_FMA");
    k.sector_fma = sf ? atoi(sf) != 0 : true;
    const char *un = getenv("GF_UNIT_NT");
    k.unit_nt = (un && atoi(un) == 128) ? 128 : 256;  // measured: c5 3.87 s (256) vs 4.41 s (128)
    return k;
}

// slot geometry (physical bit positions; qubit 0 = MSB) shared by plan
// creation and the host-only layout query
static int build_slots(gf_plan *p, int k, int sector, int n_slots, const int32_t *t1, const int32_t *t2,
                       const int32_t *logical, int n_logical)
{
    for (int s = 0; s < n_slots; ++s) {
        int a = t1[s], b = t2[s];
        if (a == b || a < 0 || b < 0 || a >= k || b >= k)
            return gf_fail(GF_EINVAL, "invalid slot targets (%d, %d) for %d qubits", a, b, k);
        if (logical && (logical[s] < 0 || logical[s] >= n_logical))
            return gf_fail(GF_EINVAL, "slot references unknown logical gate %d", logical[s]);
        SlotInfo si;
        si.swapped = a > b;
        si.q1 = std::min(a, b);
        si.q2 = std::max(a, b);
        si.logical = logical ? logical[s] : 0;
        si.mode_c1q = (sector >= 0 && si.q2 == k - 1);
        if (si.mode_c1q) {
            si.lo = p->K - 1 - si.q1;  // compressed position of qubit q1
            si.hi = -1;
        } else {
            si.lo = p->K - 1 - si.q2;
            si.hi = p->K - 1 - si.q1;
        }
        p->slots.push_back(si);
    }
    return GF_OK;
}

extern "C" int gf_plan_create(gf_plan **out, int k, int sector, int n_slots, const int32_t *t1, const int32_t *t2,
                              const int32_t *logical, int n_logical, int64_t max_batch, int chunk_states)
{
    if (!out) return gf_fail(GF_EINVAL, "null plan pointer");
    *out = nullptr;
    if (k < 2 || k > 34) return gf_fail(GF_EINVAL, "qubit count %d out of range [2, 34]", k);
    if (sector < -1 || sector > 1) return gf_fail(GF_EINVAL, "sector must be -1, 0 or 1");
    if (n_slots < 0 || n_logical < 0 || max_batch < 1 || chunk_states < 1)
        return gf_fail(GF_EINVAL, "bad plan sizes");
    gf_plan *p = new gf_plan();
    p->k = k;
    p->sector = sector;
    p->K = sector >= 0 ? k - 1 : k;
    p->n = n_slots;
    p->nlog = n_logical;
    p->max_batch = max_batch;
    p->chunk = chunk_states;
    p->N = 1ull << p->K;
    if (p->K < 2) {
        delete p;
        return gf_fail(GF_EINVAL, "state space too small");
    }
    if (int rc = build_slots(p, k, sector, n_slots, t1, t2, logical, n_logical)) {
        delete p;
        return rc;
    }
    u64 units = p->N / 4;
    int64_t ctas = (int64_t)(units / (kThreads * 4));
    p->ctas = (int)std::max<int64_t>(1, std::min<int64_t>(ctas, 148 * 8));
    {
        const PlanKnobs kn = plan_knobs(p->K, -1);
        p->fused = p->K >= 6 && !kn.stream;
        p->fm = kn.fm;
        p->fc = kn.fc;
        p->sparse_fma = !kn.sparse_dmma;
        p->c1q_dmma = kn.c1q_dmma;
        p->pair_blocks = kn.pair_blocks;
        p->lightcone = kn.lightcone;
        // (tiles of >= 2^7 amplitudes: the kernel gives each block selector its own warps)
        p->unit_fma = kn.sector_fma && sector >= 0 && p->fm >= 7 && kn.fwm >= 7;
        p->unit_nt = kn.unit_nt;
        if (p->fused) {
            p->fwd_passes = plan_passes(p, false, kn.fwm, p->unit_fma);
            p->rev_passes = plan_passes(p, true, p->fm, p->unit_fma);
            p->asc_passes.assign(p->rev_passes.rbegin(), p->rev_passes.rend());
            for (auto &f : p->asc_passes) std::reverse(f.ps, f.ps + f.nslots);
            if (getenv("GF_DUMP_PLAN")) {  // diagnostic: per-pass local bits and slot targets
                for (int sw = 0; sw < 2; ++sw) {
                    const auto &v = sw ? p->rev_passes : p->fwd_passes;
                    for (const auto &f : v) {
                        fprintf(stderr, "%s m=%d c=%d slots:", sw ? "rev" : "fwd", f.m, f.c);
                        for (int t = 0; t < f.nslots; ++t)
                            fprintf(stderr, " %d:%d,%d", f.ps[t].mode, f.ps[t].llo, f.ps[t].lhi);
                        fprintf(stderr, "\n");
                    }
                }
            }
            int mmin = p->fm;
            if (p->fm >= 11 && p->K > 10) {
                p->rev_md = plan_passes(p, true, 10);
                p->asc_md.assign(p->rev_md.rbegin(), p->rev_md.rend());
                for (auto &f : p->asc_md) std::reverse(f.ps, f.ps + f.nslots);
                mmin = 10;
            } else if (p->unit_fma) {
                // multi-direction sweeps stay on the DMMA path: they need their own geometry
                p->rev_md = plan_passes(p, true, p->fm);
                p->asc_md.assign(p->rev_md.rbegin(), p->rev_md.rend());
                for (auto &f : p->asc_md) std::reverse(f.ps, f.ps + f.nslots);
            }
            // CTAs per vector: capacity for the smallest tiles; each launch uses
            // min(capacity, its tiles), one tile per CTA by default
            u64 ntiles = 1ull << (p->K - mmin);
            p->ctas = (int)std::max<u64>(1, std::min<u64>((u64)kn.ctas, ntiles));
        }
    }
    // workspace
    size_t vbytes = sizeof(double2) * p->N * (size_t)max_batch;
    size_t pbytes = sizeof(double) * 32 * (size_t)p->ctas * max_batch * std::max(1, n_slots);
    size_t qbytes = sizeof(double) * 32 * (size_t)max_batch * std::max(1, n_slots);
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = cudaMalloc(&p->psi, vbytes);
    if (e == cudaSuccess) e = cudaMalloc(&p->bra, vbytes);
    if (e == cudaSuccess) e = cudaMalloc(&p->aux, vbytes);
    if (e == cudaSuccess) e = cudaMalloc(&p->partD, pbytes);
    if (e == cudaSuccess) e = cudaMalloc(&p->partHd, pbytes);
    if (e == cudaSuccess) e = cudaMalloc(&p->partHa, pbytes);
    if (e == cudaSuccess) e = cudaMalloc(&p->partV, sizeof(double) * 2 * (size_t)p->ctas * max_batch);
    if (e == cudaSuccess) e = cudaMalloc(&p->qD, qbytes);
    if (e == cudaSuccess) e = cudaMalloc(&p->qHd, qbytes);
    if (e == cudaSuccess) e = cudaMalloc(&p->qHa, qbytes);
    if (e == cudaSuccess) e = cudaMalloc(&p->qV, sizeof(double) * 2 * (size_t)max_batch);
    // logical -> slot CSR
    std::vector<int> lstart(n_logical + 1, 0), lslots, sw(std::max(1, n_slots), 0);
    for (int l = 0; l < n_logical; ++l) {
        lstart[l] = (int)lslots.size();
        for (int s = 0; s < n_slots; ++s)
            if (p->slots[s].logical == l) lslots.push_back(s);
    }
    lstart[n_logical] = (int)lslots.size();
    for (int s = 0; s < n_slots; ++s) sw[s] = p->slots[s].swapped;
    if (lslots.empty()) lslots.push_back(0);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_lstart, sizeof(int) * lstart.size());
    if (e == cudaSuccess) e = cudaMalloc(&p->d_lslots, sizeof(int) * lslots.size());
    if (e == cudaSuccess) e = cudaMalloc(&p->d_swapped, sizeof(int) * sw.size());
    if (e == cudaSuccess) e = cudaMemcpy(p->d_lstart, lstart.data(), sizeof(int) * lstart.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(p->d_lslots, lslots.data(), sizeof(int) * lslots.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(p->d_swapped, sw.data(), sizeof(int) * sw.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        plan_free(p);
        delete p;
        cudaGetLastError();
        return gf_fail(e == cudaErrorMemoryAllocation ? GF_ENOMEM : GF_ECUDA, "plan workspace: %s",
                       cudaGetErrorString(e));
    }
    *out = p;
    return GF_OK;
}

extern "C" int gf_plan_set_gates(gf_plan *p, const double *mats)
{
    if (p) p->frag_dirty = true;
    if (!p || !mats) return gf_fail(GF_EINVAL, "null argument");
    p->G.resize(p->n); p->Gd.resize(p->n); p->Gt.resize(p->n); p->Gc.resize(p->n);
    p->spG.assign(p->n, 0);
    for (int s = 0; s < p->n; ++s) {
        Mat4 g = to_mat4(mats + 32 * p->slots[s].logical);
        if (p->slots[s].swapped) g = wire_swap(g);
        if (p->sector >= 0 && !parity_zeros(g))
            return gf_fail(GF_EINVAL,
                           "parity-sector evaluation needs parity-conserving gates (slot %d has off-pattern entries)", s);
        p->G[s] = g;
        p->Gt[s] = transpose(g);
        p->Gc[s] = conjugate(g);
        p->Gd[s] = conjugate(p->Gt[s]);
        p->spG[s] = parity_zeros(g);
    }
    return GF_OK;
}

// nd HVP directions [nd][n_logical][4][4] evaluated in one set of sweeps
// (the fused engine shares psi / bra across them: full-Hessian columns).
extern "C" int gf_plan_set_directions_multi(gf_plan *p, int nd, const double *zmats)
{
    if (p) p->frag_dirty = true;
    if (!p || !zmats) return gf_fail(GF_EINVAL, "null argument");
    if (nd < 1 || nd > FMAXDIR) return gf_fail(GF_EINVAL, "direction count %d outside [1, %d]", nd, FMAXDIR);
    if (nd > 1 && !p->fused) return gf_fail(GF_EINVAL, "multi-direction HVP needs the fused engine");
    if (nd > p->aux_dirs) {
        // grow the per-direction workspace (chi / v vectors and HVP partials)
        const size_t vbytes = sizeof(double2) * p->N * (size_t)p->max_batch;
        const size_t pbytes = sizeof(double) * 32 * (size_t)p->ctas * p->max_batch * std::max(1, p->n);
        const size_t qbytes = sizeof(double) * 32 * (size_t)p->max_batch * std::max(1, p->n);
        double2 *aux = nullptr;
        double *phd = nullptr, *pha = nullptr, *qhd = nullptr, *qha = nullptr;
        // release the old per-direction workspace first: at 2^31 amplitudes the
        // old and new chi / v vectors do not fit side by side
        cudaFree(p->aux); cudaFree(p->partHd); cudaFree(p->partHa); cudaFree(p->qHd); cudaFree(p->qHa);
        p->aux = nullptr; p->partHd = p->partHa = p->qHd = p->qHa = nullptr;
        p->aux_dirs = 0;
        cudaError_t e = cudaMalloc(&aux, vbytes * nd);
        if (e == cudaSuccess) e = cudaMalloc(&phd, pbytes * nd);
        if (e == cudaSuccess) e = cudaMalloc(&pha, pbytes * nd);
        if (e == cudaSuccess) e = cudaMalloc(&qhd, qbytes * nd);
        if (e == cudaSuccess) e = cudaMalloc(&qha, qbytes * nd);
        if (e != cudaSuccess) {
            cudaFree(aux); cudaFree(phd); cudaFree(pha); cudaFree(qhd); cudaFree(qha);
            cudaGetLastError();
            // restore one direction's workspace so the plan stays usable
            cudaError_t r = cudaMalloc(&p->aux, vbytes);
            if (r == cudaSuccess) r = cudaMalloc(&p->partHd, pbytes);
            if (r == cudaSuccess) r = cudaMalloc(&p->partHa, pbytes);
            if (r == cudaSuccess) r = cudaMalloc(&p->qHd, qbytes);
            if (r == cudaSuccess) r = cudaMalloc(&p->qHa, qbytes);
            if (r == cudaSuccess) p->aux_dirs = 1;
            cudaGetLastError();
            p->have_z = false;
            return gf_fail(GF_ENOMEM, "direction workspace for %d directions: %s", nd, cudaGetErrorString(e));
        }
        p->aux = aux; p->partHd = phd; p->partHa = pha; p->qHd = qhd; p->qHa = qha;
        p->aux_dirs = nd;
    }
    for (int d = 0; d < nd; ++d) {
        p->Zm[d].resize(p->n); p->Ztm[d].resize(p->n);
        p->spZm[d].assign(p->n, 0); p->nzZm[d].assign(p->n, 0);
        for (int s = 0; s < p->n; ++s) {
            Mat4 z = to_mat4(zmats + 32 * (size_t)(d * p->nlog + p->slots[s].logical));
            if (p->slots[s].swapped) z = wire_swap(z);
            if (p->sector >= 0 && !parity_zeros(z))
                return gf_fail(GF_EINVAL, "sector-compressed HVP needs parity-conserving directions (slot %d)", s);
            bool nz = false;
            for (int q = 0; q < 16; ++q) nz = nz || z.m[q].x != 0.0 || z.m[q].y != 0.0;
            p->Zm[d][s] = z;
            p->Ztm[d][s] = transpose(z);
            p->spZm[d][s] = parity_zeros(z);
            p->nzZm[d][s] = nz;
        }
    }
    p->Z = p->Zm[0];
    p->Zt = p->Ztm[0];
    p->spZ = p->spZm[0];
    p->nd = nd;
    p->have_z = true;
    return GF_OK;
}

extern "C" int gf_plan_set_directions(gf_plan *p, const double *zmats)
{
    return gf_plan_set_directions_multi(p, 1, zmats);
}

// ---------------------------------------------------------------------------
// Fused pass planning: greedy over the sweep order.  A slot joins the current
// pass if its bits fit in the local set (<= m bits) and it commutes with every
// earlier slot that was skipped (no shared qubit).  Slots acting on the
// sector's implicit qubit share a virtual qubit so they never reorder among
// themselves.
// ---------------------------------------------------------------------------
// host copies of the kernel's tile addressing (ins0u, swz)
static unsigned ins0u_host(unsigned t, int b) { return ((t >> b) << (b + 1)) | (t & ((1u << b) - 1u)); }
static unsigned swz_host(unsigned l)
{
    const unsigned x = l >> 3;
    return l ^ ((__builtin_popcount(x & 0x8Bu) & 1u) | ((__builtin_popcount(x & 0x1ADu) & 1u) << 1) |
                ((__builtin_popcount(x & 0x17Bu) & 1u) << 2));
}

struct PassChoice {
    std::vector<int> slots;    // in execution order
    unsigned long long S = 0;  // local bit set (m bits)
};

// Exact beam over local-bit sets: a pass is fixed by its local set S (the c
// low bits plus m - c others); it executes, in sweep order, every remaining
// slot whose bits lie in S and that no skipped earlier slot blocks (up to
// FMAXSLOTS).  Expands every S from the best `beam` states per depth and stops
// at the first depth that executes all slots.  Used when the sets are few
// (c2: C(13, 8) = 1287 at m = 11, c = 3) and the slots fit a 64-bit mask.
// With the light-cone rule (FusedParams::fixmask) plans of equal pass count
// differ in how much slot work their dead tiles skip: `cost` = sum over passes
// of slots x 2^-(fixed global bits), minimised among the plans of the first
// complete depth.
static bool plan_exact(const gf_plan *p, const std::vector<int> &order, int m, int c, int max_depth,
                       std::vector<PassChoice> &out, bool reverse)
{
    const int n = (int)order.size(), K = p->K, nf = K - c, kf = m - c;
    if (n > 64 || nf > 40 || kf < 0 || kf > nf) return false;
    double comb = 1.0;
    for (int i = 0; i < kf; ++i) comb = comb * (nf - i) / (i + 1);
    if (comb > 20000.0) return false;
    const int VIRT = 63;
    std::vector<unsigned long long> bits(n), dep(n);
    for (int t = 0; t < n; ++t) {
        const SlotInfo &si = p->slots[order[t]];
        bits[t] = si.mode_c1q ? (1ull << si.lo) : ((1ull << si.lo) | (1ull << si.hi));
        dep[t] = bits[t] | (si.mode_c1q ? (1ull << VIRT) : 0ull);
    }
    std::vector<unsigned long long> sets;
    const unsigned long long low = (1ull << c) - 1ull;
    if (kf == 0) {
        sets.push_back(low);
    } else {
        for (unsigned long long x = (1ull << kf) - 1ull; x < (1ull << nf);) {
            sets.push_back(low | (x << c));
            const unsigned long long u = x & (~x + 1ull), v = x + u;  // Gosper's hack
            x = v + (((v ^ x) / u) >> 2);
        }
    }
    auto execute = [&](unsigned long long done, unsigned long long S) {
        unsigned long long blocked = 0ull, taken = 0ull;
        int cnt = 0;
        for (int t = 0; t < n; ++t) {
            if ((done >> t) & 1ull) continue;
            if (dep[t] & blocked) {
                blocked |= dep[t];
                continue;
            }
            if (!(bits[t] & ~S) && cnt < FMAXSLOTS) {
                taken |= 1ull << t;
                ++cnt;
            } else {
                blocked |= dep[t];
            }
        }
        return taken;
    };
    const unsigned long long all = n == 64 ? ~0ull : ((1ull << n) - 1ull);
    struct St {
        unsigned long long done;
        double cost;
        std::vector<std::pair<unsigned long long, unsigned long long>> hist;  // (taken, S)
    };
    const unsigned long long allbits = K >= 64 ? ~0ull : ((1ull << K) - 1ull);
    // slot work of a pass weighted by its live-tile fraction
    auto pass_cost = [&](unsigned long long done, unsigned long long tk, unsigned long long S) {
        if (!p->lightcone) return (double)__builtin_popcountll(tk) + 1.0;
        unsigned long long applied = 0ull;
        for (int t = 0; t < n; ++t) {
            const bool is_done = (done >> t) & 1ull;
            // forward: slots of the earlier passes; reverse: every slot not yet undone (this pass included)
            if (reverse ? !is_done : is_done) applied |= bits[t];
        }
        const int fixed = __builtin_popcountll(~S & allbits & ~applied);
        // + the pass's tile round trip on its live tiles, in slot equivalents
        return (__builtin_popcountll(tk) + 1.0) * std::ldexp(1.0, -fixed);
    };
    const size_t beam = 1500;
    typedef std::vector<std::pair<unsigned long long, unsigned long long>> Hist;
    // mode 0: fewest passes (states ranked by slots done, then cost; stops at the
    // first complete depth).  mode 1: cheapest plan within `limit` passes, ranked
    // by cost plus a guess for the slots still to run -- with dead tiles for
    // free, one more pass near the |j> end can cost less than a fuller live one.
    auto search = [&](int mode, int limit, double &best_cost, Hist &best_hist) {
        bool found = false;
        std::vector<St> cur(1);
        cur[0].done = 0ull;
        cur[0].cost = 0.0;
        for (int depth = 1; depth <= limit; ++depth) {
            std::map<unsigned long long, size_t> seen;
            std::vector<St> nxt;
            for (const St &s : cur) {
                for (unsigned long long S : sets) {
                    const unsigned long long tk = execute(s.done, S);
                    if (!tk) continue;
                    const unsigned long long nd = s.done | tk;
                    const double cost = s.cost + pass_cost(s.done, tk, S);
                    if (nd == all) {  // complete: keep the cheapest, nothing to expand
                        if (!found || cost < best_cost - 1e-12) {
                            found = true;
                            best_cost = cost;
                            best_hist = s.hist;
                            best_hist.push_back({tk, S});
                        }
                        continue;
                    }
                    auto it = seen.find(nd);
                    if (it != seen.end()) {
                        St &o = nxt[it->second];
                        if (cost < o.cost - 1e-12) {  // same slots done, cheaper passes
                            o.cost = cost;
                            o.hist = s.hist;
                            o.hist.push_back({tk, S});
                        }
                        continue;
                    }
                    seen[nd] = nxt.size();
                    St e;
                    e.done = nd;
                    e.cost = cost;
                    e.hist = s.hist;
                    e.hist.push_back({tk, S});
                    nxt.push_back(std::move(e));
                }
            }
            if (found && mode == 0) return true;
            if (nxt.empty()) break;
            std::stable_sort(nxt.begin(), nxt.end(), [&](const St &a, const St &b) {
                const int pa = __builtin_popcountll(a.done), pb = __builtin_popcountll(b.done);
                if (mode == 0) {
                    if (pa != pb) return pa > pb;
                    if (a.cost != b.cost) return a.cost < b.cost;
                    return a.done < b.done;
                }
                const double ka = a.cost + 0.6 * (n - pa), kb = b.cost + 0.6 * (n - pb);
                if (ka != kb) return ka < kb;
                return a.done < b.done;
            });
            if (nxt.size() > beam) nxt.resize(beam);
            cur.swap(nxt);
        }
        return found;
    };
    double cost0 = 0.0, cost1 = 0.0;
    Hist h0, h1;
    if (!search(0, max_depth, cost0, h0)) return false;
    const Hist *pick = &h0;
    if (p->lightcone && !getenv("GF_PLAN_MINPASS")) {
        // up to GF_PLAN_EXTRA (default 1) passes more than the minimum, if that is cheaper
        const char *xe = getenv("GF_PLAN_EXTRA");
        const int extra = xe ? std::max(0, atoi(xe)) : 1;
        if (extra > 0 && search(1, (int)h0.size() + extra, cost1, h1) && cost1 < cost0 - 1e-9) pick = &h1;
    }
    out.clear();
    for (const auto &h : *pick) {
        PassChoice pc;
        pc.S = h.second;
        for (int t = 0; t < n; ++t)
            if ((h.first >> t) & 1ull) pc.slots.push_back(order[t]);
        out.push_back(pc);
    }
    return true;
}

// PM_UNIT geometry: the unit-index columns of a slot.  col[0] is the block
// selector's column (warp-uniform in the kernel); col[1..3] (lane bits 0..2:
// one quarter-warp of a 128-bit access) are chosen linearly independent modulo
// the eight 16-byte slots of a 128-byte bank row.
static void unit_columns(PassSlot &ps, int m, bool c1q)
{
    std::vector<unsigned> cols;
    auto indep = [](unsigned a, unsigned b, unsigned c) {
        a &= 7u; b &= 7u; c &= 7u;
        return a && b && c && (a ^ b) && (a ^ c) && (b ^ c) && (a ^ b ^ c);
    };
    memset(ps.col, 0, sizeof ps.col);
    unsigned c0;
    if (!c1q) {
        for (int i = 0; i < m - 2; ++i) cols.push_back(swz_host(ins0u_host(ins0u_host(1u << i, ps.llo), ps.lhi)));
        const unsigned so = swz_host(1u << ps.llo), sh = swz_host(1u << ps.lhi);
        c0 = so;
        ps.so = so ^ sh;  // a1 = a0 ^ (so ^ sh): {00, 11} for b = 0, {01, 10} for b = 1
        ps.upar = 0;
    } else {
        // unit u = (j', b): pair index 2 j' + (b ^ parity(j') ^ tile parity ^ sector), so every
        // other column carries the parity bit's column as well
        for (int i = 0; i < m - 1; ++i) cols.push_back(swz_host(ins0u_host(1u << i, ps.llo)));
        c0 = cols[0];
        cols.erase(cols.begin());
        for (unsigned &c : cols) c ^= c0;
        ps.so = swz_host(1u << ps.llo);
        ps.upar = 1;
    }
    ps.sh = 0;
    const int nc = (int)cols.size();
    int b0 = 0, b1 = 1, b2 = 2;
    bool found = false;
    for (int i = 0; i < nc && !found; ++i)
        for (int j = i + 1; j < nc && !found; ++j)
            for (int k = j + 1; k < nc && !found; ++k)
                if (indep(cols[i], cols[j], cols[k])) {
                    b0 = i; b1 = j; b2 = k; found = true;
                }
    ps.col[0] = c0;
    int n = 1;
    if (nc >= 3) {
        ps.col[n++] = cols[b0];
        ps.col[n++] = cols[b1];
        ps.col[n++] = cols[b2];
        for (int i = 0; i < nc; ++i)
            if (i != b0 && i != b1 && i != b2) ps.col[n++] = cols[i];
    } else {
        for (unsigned c : cols) ps.col[n++] = c;
    }
}

static std::vector<FusedParams> plan_passes(const gf_plan *p, bool reverse, int m, bool unit)
{
    std::vector<FusedParams> out;
    const int n = p->n, K = p->K, c = p->fc;
    std::vector<PassChoice> choice;
    {
    std::vector<int> remaining;
    for (int i = 0; i < n; ++i) remaining.push_back(reverse ? n - 1 - i : i);
    const int VIRT = 63;
    // deterministic xorshift for the randomized best-of-N pass search
    unsigned long long rs = 0x9E3779B97F4A7C15ull;
    auto rnd = [&]() {
        rs ^= rs << 13;
        rs ^= rs >> 7;
        rs ^= rs << 17;
        return (double)(rs >> 11) * (1.0 / 9007199254740992.0);
    };
    while (!remaining.empty()) {
        unsigned long long S = 0;
        std::vector<int> taken, rest;
        // trial 0 is the plain greedy pass; later trials skip eligible slots at
        // random (keeping their qubits free for later slots) -- keep the trial
        // that executes the most slots
        for (int trial = 0; trial < 256; ++trial) {
            const double skip = trial == 0 ? 0.0 : 0.5 * rnd();
            unsigned long long S1 = (1ull << c) - 1ull, blocked = 0ull;
            std::vector<int> t1, r1;
            for (int s : remaining) {
                const SlotInfo &si = p->slots[s];
                unsigned long long bits = si.mode_c1q ? (1ull << si.lo) : ((1ull << si.lo) | (1ull << si.hi));
                unsigned long long dep = bits | (si.mode_c1q ? (1ull << VIRT) : 0ull);
                if (dep & blocked) {
                    blocked |= dep;
                    r1.push_back(s);
                    continue;
                }
                unsigned long long S2 = S1 | bits;
                if (__builtin_popcountll(S2) <= m && (int)t1.size() < FMAXSLOTS && !(skip > 0.0 && rnd() < skip)) {
                    S1 = S2;
                    t1.push_back(s);
                } else {
                    blocked |= dep;
                    r1.push_back(s);
                }
            }
            if (trial == 0 || t1.size() > taken.size()) {
                taken = t1;
                rest = r1;
                S = S1;
            }
        }
        for (int b = 0; __builtin_popcountll(S) < m && b < K; ++b) S |= 1ull << b;  // pad with low bits
        PassChoice pc;
        pc.slots = taken;
        pc.S = S;
        choice.push_back(pc);
        remaining = rest;
    }
    }
    // fewer passes (fewer tile round trips and launches) from the exact search
    // when it is affordable
    {
        std::vector<int> order;
        for (int i = 0; i < n; ++i) order.push_back(reverse ? n - 1 - i : i);
        std::vector<PassChoice> ex;
        if (choice.size() > 1 && !getenv("GF_PLAN_GREEDY") &&
            plan_exact(p, order, m, c, (int)choice.size() - (p->lightcone ? 0 : 1), ex, reverse))
            choice = ex;
    }
    for (const PassChoice &pc : choice) {
        const std::vector<int> &taken = pc.slots;
        const unsigned long long S = pc.S;
        FusedParams fp;
        memset(&fp, 0, sizeof fp);
        fp.m = m;
        fp.c = c;
        int li = 0, gi = 0;
        int lidx[64];
        for (int b = 0; b < K; ++b) {
            if ((S >> b) & 1ull) {
                lidx[b] = li;
                fp.lpos[li++] = b;
            } else {
                fp.gpos[gi++] = b;
            }
        }
        fp.nglob = gi;
        fp.ntiles = 1ull << gi;
        fp.nslots = (int)taken.size();
        for (int t = 0; t < fp.nslots; ++t) {
            const SlotInfo &si = p->slots[taken[t]];
            PassSlot ps;
            memset(&ps, 0, sizeof ps);
            ps.slot = taken[t];
            ps.mode = si.mode_c1q ? (p->c1q_dmma ? PM_C1QD : PM_C1Q) : PM_DENSE;  // sparse decided per eval
            ps.llo = lidx[si.lo];
            ps.lhi = si.mode_c1q ? 0 : lidx[si.hi];
            if (unit) {
                ps.mode = PM_UNIT;
                unit_columns(ps, m, si.mode_c1q != 0);
            } else if (ps.mode == PM_C1QD) {
                // virtual partner bit: any other local bit (the lowest one)
                const int vb = ps.llo == 0 ? 1 : 0, a0 = std::min(ps.llo, vb), a1 = std::max(ps.llo, vb);
                ps.lhi = vb;
                for (int i = 0; i < FMAXM - 1; ++i) ps.col[i] = swz_host(ins0u_host(ins0u_host(1u << i, a0), a1));
                ps.so = swz_host(1u << ps.llo);
                ps.sh = swz_host(1u << vb);
            } else if (!si.mode_c1q) {
                for (int i = 0; i < FMAXM - 1; ++i)
                    ps.col[i] = swz_host(ins0u_host(ins0u_host(1u << i, ps.llo), ps.lhi));
                ps.so = swz_host(1u << ps.llo);
                ps.sh = swz_host(1u << ps.lhi);
            } else {  // pair index -> swizzled tile index of the pair's low member
                for (int i = 0; i < FMAXM - 1; ++i) ps.col[i] = swz_host(ins0u_host(1u << i, ps.llo));
                ps.so = swz_host(1u << ps.llo);
                ps.sh = 0;
            }
            fp.ps[t] = ps;
        }
        out.push_back(fp);
    }
    // Light cone of the basis state: psi (and the forward tangent v) entering a
    // pass equal |j> on every qubit no applied slot has touched, so tiles whose
    // global bits disagree with j on such a qubit are zero (k_fused skips the
    // psi / v work there).  Forward sweep: slots of the earlier passes are
    // applied.  Reverse sweep (psi is un-computed pass by pass): the slots of
    // this and the later passes are still applied; the ascending sweep replays
    // the reverse passes backwards and sees the same set.
    if (p->lightcone) {
        auto slot_mask = [&](int s) {
            const SlotInfo &si = p->slots[s];
            return si.mode_c1q ? (1ull << si.lo) : ((1ull << si.lo) | (1ull << si.hi));
        };
        const size_t np = out.size();
        std::vector<unsigned long long> touched(np + 1, 0ull);  // by the passes' own slots
        for (size_t i = 0; i < np; ++i)
            for (int t = 0; t < out[i].nslots; ++t) touched[i] |= slot_mask(out[i].ps[t].slot);
        for (size_t i = 0; i < np; ++i) {
            unsigned long long applied = 0ull, gmask = 0ull;
            if (!reverse) {
                for (size_t j = 0; j < i; ++j) applied |= touched[j];
            } else {
                for (size_t j = i; j < np; ++j) applied |= touched[j];
            }
            for (int g = 0; g < out[i].nglob; ++g) gmask |= 1ull << out[i].gpos[g];
            out[i].fixmask = gmask & ~applied;
        }
    }
    return out;
}

static size_t fused_smem(int nv, int m, int c, int nw, int nd = 1, bool unit = false)
{
    if (unit)  // tiles, fold scratch [2][2][nw][8], global offsets, per-(slot, thread) unit bases
        return sizeof(double2) * ((size_t)nv << m) + sizeof(double) * (2 * 2 * nw * 8) +
               sizeof(unsigned long long) * ((size_t)1 << (m - c)) + sizeof(unsigned short) * FMAXSLOTS * nw * 32;
    return sizeof(double2) * ((size_t)nv << m) + sizeof(double) * ((1 + nd) * nw * 64) +
           sizeof(unsigned long long) * ((size_t)1 << (m - c));
}

template <int OP, bool FIRST, int NT, int ND, int VAR>
static int launch_fused_nt(const gf_plan *p, FusedParams &fp, int64_t nvec, cudaStream_t st)
{
    const int nv = (OP == OP_FWD || OP == OP_FWD_DOT) ? 1 : (OP == OP_REV_G ? 2 : 2 + ND);
    const size_t smem = fused_smem(nv, fp.m, fp.c, NT / 32, ND, VAR == 4);
    // the attribute is per device: set it once for every device this process drives
    static unsigned long long attr_done = 0ull;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return gf_fail(GF_ECUDA, "no current CUDA device");
    if (!((attr_done >> (dev & 63)) & 1ull)) {
        // 226 KB: the opt-in limit (227 KB) minus the kernel's static shared memory
        cudaError_t ae = cudaFuncSetAttribute(k_fused<OP, FIRST, NT, ND, VAR>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
        if (ae != cudaSuccess) return gf_fail(GF_ECUDA, "k_fused smem attribute: %s", cudaGetErrorString(ae));
        attr_done |= 1ull << (dev & 63);
    }
    if (smem > 226 * 1024) return gf_fail(GF_EINVAL, "fused tile needs %zu B of shared memory", smem);
    dim3 grid(fp.ctas, (unsigned)nvec);
    k_fused<OP, FIRST, NT, ND, VAR><<<grid, NT, smem, st>>>(fp);
    return GF_OK;
}

// 256 threads (2 CTAs/SM) for tiles up to 2^11; 512 threads (1 CTA/SM, same 16
// warps per SM) for 2^12 tiles and for multi-direction HVP sweeps (2 + ND
// vectors per tile)
template <int OP, bool FIRST, int VAR>
static int launch_fused_sp(const gf_plan *p, FusedParams &fp, int64_t nvec, cudaStream_t st, int nd)
{
    if constexpr (OP == OP_REV_GH || OP == OP_REV_H || OP == OP_ASC_H) {
        if (nd >= 2) {
            if (fp.m <= 10) {  // 2^10 tiles: 2 + ND vectors fit 2 CTAs/SM at 256 threads
                if (nd == 2) return launch_fused_nt<OP, FIRST, 256, 2, VAR>(p, fp, nvec, st);
                return launch_fused_nt<OP, FIRST, 256, 3, VAR>(p, fp, nvec, st);
            }
            if (nd == 2) return launch_fused_nt<OP, FIRST, 512, 2, VAR>(p, fp, nvec, st);
            return launch_fused_nt<OP, FIRST, 512, 3, VAR>(p, fp, nvec, st);
        }
    }
    if (fp.m >= 12 || (GF_NT512_M11 && fp.m == 11)) return launch_fused_nt<OP, FIRST, 512, 1, VAR>(p, fp, nvec, st);
    return launch_fused_nt<OP, FIRST, 256, 1, VAR>(p, fp, nvec, st);
}

template <int OP, bool FIRST>
static int launch_fused(const gf_plan *p, FusedParams &fp, int64_t nvec, cudaStream_t st, int nd = 1)
{
    bool spx = false, c1d = false, unit = fp.nslots > 0;
    for (int t = 0; t < fp.nslots; ++t) {
        // the FMA forms kept for experiments (GF_SPARSE_DMMA=0, GF_C1Q_DMMA=0) have no dead-tile variant
        if (fp.ps[t].mode == PM_SPARSE || fp.ps[t].mode == PM_C1Q) fp.fixmask = 0ull;
        spx |= (fp.ps[t].mode == PM_SPARSE);
        c1d |= (fp.ps[t].mode == PM_C1QD) || fp.ps[t].pair;
        unit = unit && (fp.ps[t].mode == PM_UNIT);
    }
    if (unit) {
        // parity-structured pass on the FMA pipe (one direction); tiles of 2^12
        // amplitudes keep the 512-thread shape
        if (nd != 1) return gf_fail(GF_EINVAL, "unit passes carry one direction");
        if (fp.m >= 12 && !(OP == OP_FWD || OP == OP_FWD_DOT))
            return launch_fused_nt<OP, FIRST, 512, 1, 4>(p, fp, nvec, st);
        if (p->unit_nt == 256) return launch_fused_nt<OP, FIRST, 256, 1, 4>(p, fp, nvec, st);
        return launch_fused_nt<OP, FIRST, 128, 1, 4>(p, fp, nvec, st);
    }
    switch ((spx ? 1 : 0) | (c1d ? 2 : 0)) {
        case 1: return launch_fused_sp<OP, FIRST, 1>(p, fp, nvec, st, nd);
        case 2: return launch_fused_sp<OP, FIRST, 2>(p, fp, nvec, st, nd);
        case 3: return launch_fused_sp<OP, FIRST, 3>(p, fp, nvec, st, nd);
        default: return launch_fused_sp<OP, FIRST, 0>(p, fp, nvec, st, nd);
    }
}

static int collect_phases(gf_plan *p);

template <int OP, bool FIRST>
static void launch_sweep(const gf_plan *p, const SlotInfo &si, bool sparse, SweepParams &sp, int64_t nvec,
                         cudaStream_t st)
{
    dim3 grid(p->ctas, (unsigned)nvec);
    if (si.mode_c1q) {
        sp.nunits = p->N / 2;
        k_sweep<OP, MODE_C1Q, FIRST><<<grid, kThreads, 0, st>>>(sp);
    } else {
        sp.nunits = p->N / 4;
        if (sparse)
            k_sweep<OP, MODE_SPARSE, FIRST><<<grid, kThreads, 0, st>>>(sp);
        else
            k_sweep<OP, MODE_DENSE, FIRST><<<grid, kThreads, 0, st>>>(sp);
    }
}

extern "C" int gf_plan_eval(gf_plan *p, int flags, int64_t nvec, const int64_t *basis, const double *weights,
                            const void *phi0, double *out, void *stream)
{
    if (!p) return gf_fail(GF_EINVAL, "null plan");
    if (nvec < 1 || nvec > p->max_batch)
        return gf_fail(GF_EINVAL, "batch of %lld summands outside [1, %lld]", (long long)nvec, (long long)p->max_batch);
    if (!basis || !phi0 || !out) return gf_fail(GF_EINVAL, "null device buffer");
    if (p->G.size() != (size_t)p->n) return gf_fail(GF_EINVAL, "gates not set");
    if ((flags & GF_HVP) && !p->have_z) return gf_fail(GF_EINVAL, "HVP requested but no directions set");
    if (!(flags & (GF_VALUE | GF_GRAD | GF_HVP))) return gf_fail(GF_EINVAL, "empty flags");
    cudaStream_t st = (cudaStream_t)stream;
    const int n = p->n;
    const int nd = (flags & GF_HVP) ? p->nd : 1;
    if (nd > 1 && !p->fused) return gf_fail(GF_EINVAL, "multi-direction HVP needs the fused engine");
    int64_t launches = 0;
    SweepParams sp;
    memset(&sp, 0, sizeof sp);
    sp.psi = p->psi;
    sp.bra = p->bra;
    sp.aux = p->aux;
    sp.phi0 = (const double2 *)phi0;
    sp.weights = weights;
    sp.N = p->N;
    sp.sector = p->sector < 0 ? 0 : p->sector;
    const size_t pstride = (size_t)32 * p->ctas * nvec;

    if (p->profiling) {
        if (p->ev_used >= 4096) collect_phases(p);
        if (p->ev_used == p->evsets.size()) {
            gf_plan::EvSet es;
            for (auto &e : es.ev) GF_CUDA(cudaEventCreate(&e));
            GF_CUDA(cudaEventCreate(&es.rev1));
            es.has_rev1 = false;
            p->evsets.push_back(es);
        }
        gf_plan::EvSet &es = p->evsets[p->ev_used++];
        es.has_rev1 = false;
        for (int i = 0; i < 5; ++i) p->ev[i] = es.ev[i];
        p->ev_rev1 = es.rev1;
        p->pending = 1;
        GF_CUDA(cudaEventRecord(p->ev[0], st));
    }
    if (!(p->fused && n > 0)) {
        u64 total = p->N * (u64)nvec;
        int blocks = (int)std::min<u64>((total + 255) / 256, 148 * 16);
        k_init_basis<<<blocks, 256, 0, st>>>(p->psi, p->N, basis, nvec);
        ++launches;
    }
    int64_t l_fwd = 0, l_rev = 0, l_asc = 0;
    int ctas_r = p->ctas, ctas_v = p->ctas;  // CTAs per vector of the hole / value partials
    const bool grad_like = (flags & (GF_GRAD | GF_HVP)) != 0;
    if (n == 0) {
        // empty circuit: value = sum phi0 . |j>; an identity "slot" with the dot fused
        Mat4 I;
        for (int e = 0; e < 16; ++e) I.m[e] = make_double2((e % 5 == 0) ? 1.0 : 0.0, 0.0);
        SlotInfo si;
        si.q1 = 0; si.q2 = 1; si.swapped = false; si.logical = 0; si.mode_c1q = 0; si.lo = 0; si.hi = 1;
        sp.lo = 0; sp.hi = 1; sp.A = I; sp.partV = p->partV;
        launch_sweep<OP_FWD_DOT, false>(p, si, false, sp, nvec, st);
        ++launches;
    }
    if (p->fused && n > 0) {
        FusedParams fp;
        static const bool exp_noslots = getenv("GF_EXP_NOSLOTS") != nullptr;  // timing diagnostic only
        if (int rc_ = upload_frags(p, st)) return rc_;
        auto setup = [&](FusedParams &f) {
            f.frag = p->d_frag;
            f.psi = p->psi;
            f.bra = p->bra;
            f.aux = p->aux;
            f.phi0 = (const double2 *)phi0;
            f.weights = weights;
            f.N = p->N;
            f.nvec = (int)nvec;
            f.ctas = (int)std::min<u64>((u64)p->ctas, f.ntiles);
            f.sector = p->sector < 0 ? 0 : p->sector;
            f.partV = p->partV;
            f.qV = p->qV;
            f.basis = basis;
            f.store_mask = 7;
            f.auxstride = p->N * (u64)p->max_batch;
            f.hstride = (u64)std::max(1, p->n) * p->max_batch * p->ctas * 32;
            f.qhstride = (u64)std::max(1, p->n) * p->max_batch * 32;
            if (exp_noslots) f.nslots = 0;
            static const bool exp_noio = getenv("GF_EXP_NOIO") != nullptr;  // timing diagnostic only
            f.exp_noio = exp_noio ? 1 : 0;
        };
        const bool md = nd >= 2 && !p->rev_md.empty() && (flags & GF_HVP);
        const std::vector<FusedParams> &revp = md ? p->rev_md : p->rev_passes;
        const std::vector<FusedParams> &ascp = md ? p->asc_md : p->asc_passes;
        const int nf = (int)p->fwd_passes.size(), nr = (int)revp.size();
        for (int pi = 0; pi < nf; ++pi) {
            fp = p->fwd_passes[pi];
            setup(fp);
            for (int t = 0; t < fp.nslots; ++t) {
                const int s = fp.ps[t].slot;
                fp.mat[t][0] = p->G[s];
                fp.ps[t].fa = s * NFK + FK_G;
                fp.ps[t].fa2 = fp.ps[t].fa;
                fp.ps[t].fb = fp.ps[t].fa;
                fp.ps[t].fz = fp.ps[t].fa;
                if (fp.ps[t].mode != PM_C1Q && fp.ps[t].mode != PM_C1QD && fp.ps[t].mode != PM_UNIT) fp.ps[t].mode = (p->spG[s] && p->sparse_fma) ? PM_SPARSE : PM_DENSE;
            }
            const bool last = !grad_like && pi == nf - 1;
            if (last) ctas_v = fp.ctas;
            if (pi == 0) {
                if (last) fp.store_mask = 0;  // value only: psi_n is not needed afterwards
                if (last) { int rc_ = launch_fused<OP_FWD_DOT, true>(p, fp, nvec, st); if (rc_) return rc_; }
                else { int rc_ = launch_fused<OP_FWD, true>(p, fp, nvec, st); if (rc_) return rc_; }
            } else {
                if (last) { int rc_ = launch_fused<OP_FWD_DOT, false>(p, fp, nvec, st); if (rc_) return rc_; }
                else { int rc_ = launch_fused<OP_FWD, false>(p, fp, nvec, st); if (rc_) return rc_; }
            }
            ++launches;
        }
        l_fwd = launches;
        if (p->profiling) GF_CUDA(cudaEventRecord(p->ev[1], st));
        if (grad_like) {
            const bool h = (flags & GF_HVP) != 0;
            int act_rev = 0;  // directions whose chi is nonzero entering the next slot
            for (int pi = 0; pi < nr; ++pi) {
                fp = revp[pi];
                setup(fp);
                ctas_r = fp.ctas;
                if (pi == 0) ctas_v = fp.ctas;
                fp.partD = p->partD;
                fp.partH = p->partHd;
                fp.qD = p->qD;
                fp.qH = p->qHd;
                for (int t = 0; t < fp.nslots; ++t) {
                    const int s = fp.ps[t].slot;
                    fp.mat[t][0] = p->Gd[s];
                    fp.mat[t][1] = p->Gt[s];
                    fp.ps[t].fa = s * NFK + FK_GD;
                    fp.ps[t].fa2 = s * NFK + FK_GDA;
                    fp.ps[t].fb = s * NFK + FK_GT;
                    fp.ps[t].fz = s * NFK + FK_ZT;
                    bool sp = p->spG[s];
                    fp.ps[t].zmask = 0;
                    if (h) {
                        for (int d = 0; d < nd; ++d) {
                            fp.mat[t][2 + d] = p->Ztm[d][s];
                            sp = sp && p->spZm[d][s];
                            fp.ps[t].zmask |= p->nzZm[d][s] ? (1 << d) : 0;
                        }
                    }
                    fp.ps[t].amask = act_rev;
                    act_rev |= fp.ps[t].zmask;
                    if (fp.ps[t].mode != PM_C1Q && fp.ps[t].mode != PM_C1QD && fp.ps[t].mode != PM_UNIT) fp.ps[t].mode = (sp && p->sparse_fma) ? PM_SPARSE : PM_DENSE;
                    // paired parity blocks: one direction, parity-structured G and Z on the DMMA path
                    fp.ps[t].pair = h && nd == 1 && p->pair_blocks &&
                                    (fp.ps[t].mode == PM_C1QD || (fp.ps[t].mode == PM_DENSE && sp));
                    fp.ps[t].pblk = fp.ps[t].mode == PM_C1QD ? 1 : 0;
                    fp.ps[t].fpe = s * NFK + FK_PRE;
                }
                // after the reverse sweep psi_0 = |j> is known exactly and chi is dead:
                // the last pass writes back only the bra (needed by the ascending sweep)
                if (pi == nr - 1) fp.store_mask = h ? 2 : 0;
                if (h) {
                    // HVP-only evaluations skip the gradient hole
                    const bool g = (flags & GF_GRAD) != 0;
                    int rc_;
                    if (pi == 0) rc_ = g ? launch_fused<OP_REV_GH, true>(p, fp, nvec, st, nd)
                                         : launch_fused<OP_REV_H, true>(p, fp, nvec, st, nd);
                    else rc_ = g ? launch_fused<OP_REV_GH, false>(p, fp, nvec, st, nd)
                                 : launch_fused<OP_REV_H, false>(p, fp, nvec, st, nd);
                    if (rc_) return rc_;
                } else {
                    if (pi == 0) { int rc_ = launch_fused<OP_REV_G, true>(p, fp, nvec, st); if (rc_) return rc_; }
                    else { int rc_ = launch_fused<OP_REV_G, false>(p, fp, nvec, st); if (rc_) return rc_; }
                }
                if (pi == 0 && p->profiling && p->ev_rev1) {
                    GF_CUDA(cudaEventRecord(p->ev_rev1, st));
                    p->evsets[p->ev_used - 1].has_rev1 = true;
                    p->rev1_slots = fp.nslots;
                    p->rev1_vectors += nvec;
                    p->rev1_launches += 1;
                }
                ++launches;
            }
            l_rev = launches - l_fwd;
            if (p->profiling) GF_CUDA(cudaEventRecord(p->ev[2], st));
            if (h) {
                int act_asc = 0;  // directions whose v is nonzero entering the next slot
                for (int pi = 0; pi < nr; ++pi) {
                    fp = ascp[pi];
                    setup(fp);
                    fp.partH = p->partHa;
                    fp.qH = p->qHa;
                    for (int t = 0; t < fp.nslots; ++t) {
                        const int s = fp.ps[t].slot;
                        fp.mat[t][0] = p->Gc[s];
                        fp.mat[t][1] = p->G[s];
                        fp.ps[t].fa = s * NFK + FK_GC;
                        fp.ps[t].fa2 = s * NFK + FK_GCA;
                        fp.ps[t].fb = s * NFK + FK_G;
                        fp.ps[t].fz = s * NFK + FK_Z;
                        bool sp = p->spG[s];
                        fp.ps[t].zmask = 0;
                        for (int d = 0; d < nd; ++d) {
                            fp.mat[t][2 + d] = p->Zm[d][s];
                            sp = sp && p->spZm[d][s];
                            fp.ps[t].zmask |= p->nzZm[d][s] ? (1 << d) : 0;
                        }
                        fp.ps[t].amask = act_asc;
                        act_asc |= fp.ps[t].zmask;
                        if (fp.ps[t].mode != PM_C1Q && fp.ps[t].mode != PM_C1QD && fp.ps[t].mode != PM_UNIT) fp.ps[t].mode = (sp && p->sparse_fma) ? PM_SPARSE : PM_DENSE;
                        fp.ps[t].pair = nd == 1 && p->pair_blocks &&
                                        (fp.ps[t].mode == PM_C1QD || (fp.ps[t].mode == PM_DENSE && sp));
                        fp.ps[t].pblk = fp.ps[t].mode == PM_C1QD ? 1 : 0;
                        fp.ps[t].fpe = s * NFK + FK_PAE;
                    }
                    if (pi == nr - 1) fp.store_mask = 0;  // nothing is read after the ascending sweep
                    if (pi == 0) { int rc_ = launch_fused<OP_ASC_H, true>(p, fp, nvec, st, nd); if (rc_) return rc_; }
                    else { int rc_ = launch_fused<OP_ASC_H, false>(p, fp, nvec, st, nd); if (rc_) return rc_; }
                    ++launches;
                }
            }
        }
    } else {
    // forward sweep
        for (int s = 0; s < n; ++s) {
            const SlotInfo &si = p->slots[s];
            sp.lo = si.lo;
            sp.hi = si.hi;
            sp.A = p->G[s];
            if (!grad_like && s == n - 1) {
                sp.partV = p->partV;
                launch_sweep<OP_FWD_DOT, false>(p, si, p->spG[s], sp, nvec, st);
            } else {
                launch_sweep<OP_FWD, false>(p, si, p->spG[s], sp, nvec, st);
            }
            ++launches;
        }
        l_fwd = launches;
        if (p->profiling) GF_CUDA(cudaEventRecord(p->ev[1], st));
        if (grad_like && n > 0) {
            const bool h = (flags & GF_HVP) != 0;
            for (int s = n - 1; s >= 0; --s) {
                const SlotInfo &si = p->slots[s];
                sp.lo = si.lo;
                sp.hi = si.hi;
                sp.A = p->Gd[s];
                sp.B = p->Gt[s];
                sp.partD = p->partD + pstride * s;
                sp.partV = p->partV;
                const bool first = (s == n - 1);
                if (h) {
                    sp.C = p->Zt[s];
                    sp.partH = p->partHd + pstride * s;
                    bool sparse = p->spG[s] && p->spZ[s];
                    if (first) launch_sweep<OP_REV_GH, true>(p, si, sparse, sp, nvec, st);
                    else launch_sweep<OP_REV_GH, false>(p, si, sparse, sp, nvec, st);
                } else {
                    if (first) launch_sweep<OP_REV_G, true>(p, si, p->spG[s], sp, nvec, st);
                    else launch_sweep<OP_REV_G, false>(p, si, p->spG[s], sp, nvec, st);
                }
                ++launches;
            }
            l_rev = launches - l_fwd;
            if (p->profiling) GF_CUDA(cudaEventRecord(p->ev[2], st));
            if (h) {
                for (int s = 0; s < n; ++s) {
                    const SlotInfo &si = p->slots[s];
                    sp.lo = si.lo;
                    sp.hi = si.hi;
                    sp.A = p->Gc[s];
                    sp.B = p->G[s];
                    sp.C = p->Z[s];
                    sp.partH = p->partHa + pstride * s;
                    bool sparse = p->spG[s] && p->spZ[s];
                    if (s == 0) launch_sweep<OP_ASC_H, true>(p, si, sparse, sp, nvec, st);
                    else launch_sweep<OP_ASC_H, false>(p, si, sparse, sp, nvec, st);
                    ++launches;
                }
            }
        }
    }
    if (!(grad_like && n > 0) && p->profiling) GF_CUDA(cudaEventRecord(p->ev[2], st));
    l_asc = launches - l_fwd - l_rev;
    if (p->profiling) GF_CUDA(cudaEventRecord(p->ev[3], st));
    if (grad_like && n > 0) {
        int64_t nsb = (int64_t)n * nvec;
        int blocks = (int)((nsb * 32 + 255) / 256);
        if (flags & GF_GRAD) {  // HVP-only evaluations write no gradient partials
            k_reduce_ctas<<<blocks, 256, 0, st>>>(p->partD, p->qD, nsb, ctas_r);
            ++launches;
        }
        if (flags & GF_HVP) {
            const int ndr = p->fused ? nd : 1;
            const u64 hs = (u64)std::max(1, p->n) * p->max_batch * p->ctas * 32;
            const u64 qs = (u64)std::max(1, p->n) * p->max_batch * 32;
            for (int d = 0; d < ndr; ++d) {
                k_reduce_ctas<<<blocks, 256, 0, st>>>(p->partHd + d * hs, p->qHd + d * qs, nsb, ctas_r);
                k_reduce_ctas<<<blocks, 256, 0, st>>>(p->partHa + d * hs, p->qHa + d * qs, nsb, ctas_r);
                launches += 2;
            }
        }
    }
    if (p->fused && n > 0) {
        k_reduce_ctas<<<(unsigned)((nvec * 2 + 255) / 256), 256, 0, st>>>(p->partV, p->qV, nvec, ctas_v, 2);
        ++launches;
    }
    {
        int64_t nchunks = (nvec + p->chunk - 1) / p->chunk;
        int rec = 2 + 32 * p->nlog * (1 + nd);
        int64_t tot = nchunks * rec;
        int eff = (n > 0) ? flags : (flags & GF_VALUE);
        const bool fusedV = p->fused && n > 0;
        k_chunk_records<<<(unsigned)((tot * 32 + 255) / 256), 256, 0, st>>>(
            p->qD, p->qHd, p->qHa, fusedV ? p->qV : p->partV, nvec, fusedV ? 1 : p->ctas, n, p->nlog, p->d_lstart,
            p->d_lslots, p->d_swapped, p->chunk, eff, p->sector >= 0, nd,
            (int64_t)std::max(1, p->n) * p->max_batch * 32, out);
        ++launches;
    }
    if (p->profiling) {
        GF_CUDA(cudaEventRecord(p->ev[4], st));
        p->phase_launches[0] += l_fwd;
        p->phase_launches[1] += l_rev;
        p->phase_launches[2] += l_asc;
        p->phase_launches[3] += launches - l_fwd - l_rev - l_asc;
    }
    GF_CUDA(cudaGetLastError());
    p->last_launches = launches;
    p->last_flags = flags;
    return GF_OK;
}

static int collect_phases(gf_plan *p)
{
    if (!p->pending || p->ev_used == 0) return GF_OK;
    GF_CUDA(cudaEventSynchronize(p->evsets[p->ev_used - 1].ev[4]));
    for (size_t k = 0; k < p->ev_used; ++k) {
        const gf_plan::EvSet &es = p->evsets[k];
        for (int i = 0; i < 4; ++i) {
            float ms = 0.f;
            GF_CUDA(cudaEventElapsedTime(&ms, es.ev[i], es.ev[i + 1]));
            p->phase_ms[i] += ms;
        }
        if (es.has_rev1) {
            float ms = 0.f;
            GF_CUDA(cudaEventElapsedTime(&ms, es.ev[1], es.rev1));
            p->rev1_ms += ms;
        }
    }
    p->ev_used = 0;
    p->pending = 0;
    return GF_OK;
}

extern "C" int gf_plan_set_profiling(gf_plan *p, int on)
{
    if (!p) return gf_fail(GF_EINVAL, "null plan");
    p->profiling = on != 0;
    p->pending = 0;
    p->ev_used = 0;
    p->rev1_pending = false;
    p->rev1_ms = 0.0;
    p->rev1_launches = p->rev1_vectors = 0;
    for (int i = 0; i < 4; ++i) {
        p->phase_ms[i] = 0.0;
        p->phase_launches[i] = 0;
    }
    return GF_OK;
}

extern "C" int gf_plan_phase_times(gf_plan *p, double *ms4, int64_t *launches4)
{
    if (!p || !ms4) return gf_fail(GF_EINVAL, "null argument");
    int rc = collect_phases(p);
    if (rc) return rc;
    for (int i = 0; i < 4; ++i) {
        ms4[i] = p->phase_ms[i];
        if (launches4) launches4[i] = p->phase_launches[i];
    }
    return GF_OK;
}

// First reverse pass of the profiled evaluations: accumulated device time,
// launches, summand vectors processed and the slots of the pass.
extern "C" int gf_plan_first_reverse_pass(gf_plan *p, double *ms, int64_t *launches, int64_t *vectors, int *slots)
{
    if (!p) return gf_fail(GF_EINVAL, "null plan");
    if (p->pending) {
        int rc = collect_phases(p);
        if (rc) return rc;
    }
    if (ms) *ms = p->rev1_ms;
    if (launches) *launches = p->rev1_launches;
    if (vectors) *vectors = p->rev1_vectors;
    if (slots) *slots = p->rev1_slots;
    return GF_OK;
}

extern "C" int gf_plan_slot_outputs(gf_plan *p, int64_t nvec, double *d_dev, double *h_dev, void *stream)
{
    if (!p || nvec < 1 || nvec > p->max_batch) return gf_fail(GF_EINVAL, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    int blocks = (p->n * 32 + 255) / 256;
    if (blocks == 0) return GF_OK;
    if (d_dev) k_slot_sums<<<blocks, 256, 0, st>>>(p->qD, nullptr, nvec, p->n, p->sector >= 0, d_dev);
    if (h_dev) k_slot_sums<<<blocks, 256, 0, st>>>(p->qHd, p->qHa, nvec, p->n, p->sector >= 0, h_dev);
    GF_CUDA(cudaGetLastError());
    return GF_OK;
}

extern "C" int64_t gf_plan_last_launches(const gf_plan *p) { return p ? p->last_launches : 0; }

extern "C" int gf_plan_destroy(gf_plan *p)
{
    if (!p) return GF_OK;
    plan_free(p);
    delete p;
    return GF_OK;
}

// Host-only: the fused pass plan the engine would use for this circuit
// (no device work).  sweep 0 = forward, 1 = reverse (the ascending sweep
// replays the reverse plan backwards).  pass_sizes[i] = slots in pass i,
// slot_order = the slots in execution order, pass_bits[i] = the pass's local
// bit set (physical positions).
extern "C" int gf_plan_layout(int k, int sector, int n_slots, const int32_t *t1, const int32_t *t2, int tile_bits,
                              int sweep, int max_passes, int *n_passes, int *pass_sizes, int *slot_order,
                              unsigned long long *pass_bits)
{
    if (!n_passes || !pass_sizes || !slot_order || !pass_bits || max_passes < 1)
        return gf_fail(GF_EINVAL, "null output or no room for passes");
    if (k < 2 || k > 34 || sector < -1 || sector > 1 || n_slots < 1)
        return gf_fail(GF_EINVAL, "bad layout query sizes");
    gf_plan tmp;
    tmp.k = k;
    tmp.sector = sector;
    tmp.K = sector >= 0 ? k - 1 : k;
    tmp.n = n_slots;
    if (int rc = build_slots(&tmp, k, sector, n_slots, t1, t2, nullptr, 0)) return rc;
    const PlanKnobs kn = plan_knobs(tmp.K, std::max(1, tile_bits));
    tmp.fm = kn.fm;
    tmp.fc = kn.fc;
    tmp.c1q_dmma = kn.c1q_dmma;
    tmp.lightcone = kn.lightcone;
    std::vector<FusedParams> passes = plan_passes(&tmp, sweep != 0, tmp.fm);
    if ((int)passes.size() > max_passes) return gf_fail(GF_EINVAL, "%zu passes exceed the output room", passes.size());
    *n_passes = (int)passes.size();
    int o = 0;
    for (size_t i = 0; i < passes.size(); ++i) {
        pass_sizes[i] = passes[i].nslots;
        unsigned long long bits = 0;
        for (int b = 0; b < passes[i].m; ++b) bits |= 1ull << passes[i].lpos[b];
        pass_bits[i] = bits;
        for (int t = 0; t < passes[i].nslots; ++t) slot_order[o++] = passes[i].ps[t].slot;
    }
    return GF_OK;
}

// Live fraction of the slot work per sweep under the light-cone rule
// (FusedParams::fixmask): sum over passes of slots x 2^-popcount(fixmask),
// divided by the slot count.  frac3 = {forward, reverse, ascending}.
extern "C" int gf_plan_live_fraction(const gf_plan *p, double *frac3)
{
    if (!p || !frac3) return gf_fail(GF_EINVAL, "null argument");
    auto frac = [&](const std::vector<FusedParams> &v) {
        double live = 0.0, tot = 0.0;
        for (const FusedParams &f : v) {
            live += f.nslots * std::ldexp(1.0, -__builtin_popcountll(f.fixmask));
            tot += f.nslots;
        }
        return tot > 0.0 ? live / tot : 1.0;
    };
    frac3[0] = p->fused ? frac(p->fwd_passes) : 1.0;
    frac3[1] = p->fused ? frac(p->rev_passes) : 1.0;
    frac3[2] = p->fused ? frac(p->asc_passes) : 1.0;
    return GF_OK;
}

extern "C" int gf_plan_describe(const gf_plan *p, int *fused, int *tile_bits, int *n_fwd_passes, int *n_rev_passes,
                                int *ctas)
{
    if (!p) return gf_fail(GF_EINVAL, "null plan");
    if (fused) *fused = p->fused ? 1 : 0;
    if (tile_bits) *tile_bits = p->fm;
    if (n_fwd_passes) *n_fwd_passes = (int)p->fwd_passes.size();
    if (n_rev_passes) *n_rev_passes = (int)p->rev_passes.size();
    if (ctas) *ctas = p->ctas;
    return GF_OK;
}
