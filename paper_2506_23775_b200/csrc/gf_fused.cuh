// gf_fused.cuh -- fused k-qubit tile passes (north-star item 1).
//
// A pass applies a run of slots whose target bits all lie in a set S of m
// "local" bit positions (always including the c = 3 lowest bits, so every HBM
// access is a >= 128 B contiguous run, one full DRAM line).  One CTA stages a
// tile -- the 2^m amplitudes sharing one assignment of the K-m global bits --
// of every vector the sweep touches (psi, bra, chi/v) in shared memory, runs
// all slots of the pass on it, and writes it back: one HBM round trip per pass
// instead of one per slot.
//
// All dense FP64 math runs on the tensor cores (DMMA m8n8k4):
//  * gate applications: a lane owns one complex amplitude of an 8-tuple group
//    and y = G x is two MMA k-steps with G's real 8x8 form as the B fragment;
//  * 4x4 hole contractions (reference kernels.py:208-242): with the complex
//    4-vectors split into 8 real components, C[r][s] = sum_env bra_r ket_s is
//    an 8x8 GEMM with the environment as K, accumulated in 2 registers per
//    lane; the warps' fragments are summed in a fixed order in shared memory,
//    so the result is deterministic.
// Parity-structured passes (parity sectors: every slot is parity conserving)
// run as FP64 FMAs on two-amplitude units instead (PM_UNIT, run_units): half
// the flops of the dense DMMA form, one shared-memory round trip per slot.
#pragma once
#include "gf_common.cuh"

namespace gf {

constexpr int FT = 256;         // threads per fused CTA (8 warps)
constexpr int FMAXM = 12;       // max local bits
constexpr int FMAXSLOTS = 16;   // max slots per pass (kernel parameter space: 16 x 5 Mat4)
constexpr int FMAXGLOB = 40;
constexpr int FMAXDIR = 3;      // HVP directions per sweep (full-Hessian columns)

// PM_UNIT: parity-structured slots (parity-conserving 2q gates and the sector's
// parity-controlled 1q gates) as FP64 FMAs on *units* -- two amplitudes plus a
// block selector b -- with the whole slot (gate, holes, updates) in registers
enum { PM_DENSE = 0, PM_SPARSE = 1, PM_C1Q = 2, PM_C1QD = 3, PM_UNIT = 4 };

// rows of the per-slot DMMA fragment table: G, G^dag, G^T, conj G, then Z_d^T
// and Z_d per direction (row = slot * NFK + kind, 32 lanes per row)
// FK_GDA / FK_GCA: G^dag and conj G as the A operand of C = G X (the fused
// gate + hole formulation of the reverse / ascending passes)
enum {
    FK_G = 0, FK_GD = 1, FK_GT = 2, FK_GC = 3, FK_ZT = 4, FK_Z = 4 + FMAXDIR,
    FK_GDA = 4 + 2 * FMAXDIR, FK_GCA = 5 + 2 * FMAXDIR,
    // paired parity-block fragments (PassSlot::pair): per block {E, O} one row
    // (x input, X input) = ([M1_b | M2_b], [0 | M1_b]) for the reverse sweep
    // (M1 = G^T, M2 = Z^T) and the ascending sweep (M1 = G, M2 = Z)
    FK_PRE = 6 + 2 * FMAXDIR, FK_PRO = 7 + 2 * FMAXDIR, FK_PAE = 8 + 2 * FMAXDIR, FK_PAO = 9 + 2 * FMAXDIR,
    NFK = 10 + 2 * FMAXDIR
};

struct PassSlot {
    int slot;  // circuit slot index (for the partial layout)
    int mode;  // PM_*
    int llo;   // local bit index of the low target bit (c1q: the explicit qubit)
    int lhi;   // local bit index of the high target bit (unused for c1q)
    int zmask; // bit d: direction d has a nonzero Z at this slot (zero Z-terms are skipped)
    int amask; // bit d: chi_d / v_d is nonzero entering this slot (else its hole and update are skipped)
    int fa, fb, fz;  // fragment-table rows of mat[0], mat[1], mat[2 + d] (fz + d)
    int fa2;         // row of mat[0] in A-operand form (fused gate + hole passes)
    int pair;        // update phase as two parity-block DMMAs per input (one direction, parity-structured G, Z)
    int fpe;         // fragment row of the even block (the odd block is fpe + 1)
    int pblk;        // block amplitudes: 0 = {0,3} / {1,2} (parity gate), 1 = {0,1} / {2,3} (PM_C1QD virtual)
    // 2q slots: col[i] = swz(tuple index 2^i with zeros inserted at llo, lhi),
    // so = swz(2^llo), sh = swz(2^lhi); c1q slots: col[i] = swz(pair index 2^i
    // with a zero inserted at llo), so = swz(2^llo) -- the GF(2)-linear tile
    // addressing, precomputed on the host instead of per slot and lane
    // PM_UNIT slots: unit index u (bit 0 = block selector b) -> swizzled tile
    // index of the unit's first amplitude a0 = XOR_i u_i col[i] (^ col[0] when
    // upar and the tile's parity ^ sector is odd); second amplitude a1 = a0 ^ so.
    // The host orders the columns so that col[0..2] are independent modulo the
    // eight 16-byte slots of a bank row (conflict-free 128-bit accesses).
    unsigned col[FMAXM - 1];
    unsigned so, sh;
    int upar;        // PM_UNIT: parity-controlled 1q slot (block selector = parity of the pair index)
};

struct FusedParams {
    double2 *psi, *bra, *aux;  // [nvec][N]
    const double2 *phi0;       // [nvec][N]
    const double *weights;     // [nvec] or null
    const int64_t *basis;      // [nvec] (first forward pass synthesises |j>)
    const double2 *frag;       // [n slots][NFK][32] per-lane DMMA B fragments (gf_plan::d_frag)
    double *partD, *partH, *partV;
    double *qD, *qH, *qV;    // per-(slot, vector) sums (k_reduce_ctas)
    unsigned long long N;
    unsigned long long ntiles;  // 2^(K-m)
    // light cone: global bit positions on which psi (and v) entering this pass
    // still equal the basis state (no applied slot has touched them); a tile
    // that disagrees with j on one of them holds psi = v = 0 (0 = disabled)
    unsigned long long fixmask;
    int nvec, ctas, sector;
    int m, c, nglob, nslots;
    int exp_noio;    // timing diagnostic (GF_EXP_NOIO): skip the tile loads and stores
    int store_mask;  // bit 0 psi, bit 1 bra, bit 2 chi/v: vectors written back after the pass
    unsigned long long auxstride; // aux (chi / v) offset between directions (amplitudes)
    unsigned long long hstride;   // partH / qH offset between directions (doubles)
    unsigned long long qhstride;
    int lpos[FMAXM];
    int gpos[FMAXGLOB];
    PassSlot ps[FMAXSLOTS];
    Mat4 mat[FMAXSLOTS][2 + FMAXDIR];  // FWD {G}; REV {G^dag, G^T, Z_d^T...}; ASC {conj G, G, Z_d...}
};

}  // namespace gf
