// culorads.cu -- sm_100a kernels for the low-rank SDP solve path (see include/culorads.h).
//
// All arithmetic is fp64. The work is HBM-bound gather/stream traffic over
// n x ld factors (no GEMM-shaped contraction exists on this path), so the
// kernels are built around: 16-byte (double2) loads of factor rows, one
// lane group per pattern/constraint row sized to the padded rank, index and
// coefficient loads done cooperatively by the group and broadcast with
// shuffles, grids sized in multiples of the 148 SMs, and deterministic
// two-level reductions (per-block partials, the last block folds them in a
// fixed order).

#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "culorads.h"

#define NT 256
#define NWARP (NT / 32)
#define NSM 148

namespace {

// ---------------------------------------------------------------------------
// deterministic reductions
// ---------------------------------------------------------------------------

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Reduce acc[0..ndot) over the block, store per-block partials, and let the
// last block to finish fold all partials (fixed order) into out[0..ndot).
// ws layout: [CL_RED_BLOCKS * CL_MAXDOT partials][1 counter word].
template <int ND>
__device__ __forceinline__ void reduce_and_finish(const double (&acc)[ND], int ndot, double* ws,
                                                  double* out, int gap_at = ND, int gap = 0) {
    __shared__ double sh[NWARP][ND > 0 ? ND : 1];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
        if (d < ndot) {
            double v = warp_sum(acc[d]);
            if (lane == 0) sh[wid][d] = v;
        }
    }
    __syncthreads();
    if (threadIdx.x < ndot) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < NWARP; ++w) s += sh[w][threadIdx.x];
        ws[(size_t)blockIdx.x * CL_MAXDOT + threadIdx.x] = s;
    }
    __threadfence();
    __syncthreads();
    unsigned int* counter = reinterpret_cast<unsigned int*>(ws + CL_WS_DOUBLES);
    if (threadIdx.x == 0) {
        unsigned int prev = atomicAdd(counter, 1u);
        last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // one warp per dot, lanes stride over the block partials
    for (int d = wid; d < ndot; d += NWARP) {
        double s = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32)
            s += __ldcg(ws + (size_t)b * CL_MAXDOT + d);
        s = warp_sum(s);
        if (lane == 0) out[d + (d >= gap_at ? gap : 0)] = s;
    }
    if (threadIdx.x == 0) *counter = 0u;
}

__device__ __forceinline__ double2 ld2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ double2 ld2cs(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }
// Explicit rounding (no compiler-chosen contraction): every kernel evaluates a 16-byte
// dot the same way, so fused and unfused paths that read the same operands agree bit for bit.
__device__ __forceinline__ double dot2(double2 a, double2 b) { return fma(a.y, b.y, __dmul_rn(a.x, b.x)); }
__device__ __forceinline__ double2 axpy2(double a, double2 x, double2 y) {
    return make_double2(fma(a, x.x, y.x), fma(a, x.y, y.y));
}

template <int K>
__device__ __forceinline__ double2 select2(const double2 (&v)[K], int idx) {
    double2 r = v[0];
#pragma unroll
    for (int j = 1; j < K; ++j)
        if (idx == j) r = v[j];
    return r;
}

int red_grid(int64_t work_items) {
    int64_t g = (work_items + NT - 1) / NT;
    if (g < 1) g = 1;
    if (g > CL_RED_BLOCKS) g = CL_RED_BLOCKS;
    return (int)g;
}

// Resident CTAs per SM of a kernel at NT threads (occupancy query, cached per kernel).
int resident_blocks(const void* fn) {
    static const void* keys[128];
    static int vals[128];
    static int cnt = 0;
    for (int i = 0; i < cnt; ++i)
        if (keys[i] == fn) return vals[i];
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, NT, 0) != cudaSuccess || nb < 1) nb = 1;
    if (cnt < 128) {
        keys[cnt] = fn;
        vals[cnt] = nb;
        ++cnt;
    }
    return nb;
}

// Grid of a grid-stride kernel: one full wave of resident CTAs (148 x CTAs/SM), fewer when
// the work is smaller -- a partial second wave would idle part of the GPU at the end.
int occ_grid(const void* fn, int64_t work_items, int64_t cap = CL_RED_BLOCKS) {
    int64_t g = (work_items + NT - 1) / NT;
    int64_t wave = (int64_t)resident_blocks(fn) * NSM;
    if (wave > cap) wave = cap;
    if (g > wave) g = wave;
    if (g < 1) g = 1;
    return (int)g;
}

// ---------------------------------------------------------------------------
// streaming combination
// ---------------------------------------------------------------------------

struct LcDev {
    int nin, ndot;
    const double* in[CL_MAXIN];
    double coef[CL_MAXIN];
    double* out;
    uint8_t da[CL_MAXDOT], db[CL_MAXDOT];
};

// MODE 0: up to 7 inputs, <= 8 arbitrary pair dots (operand 7 = out)
// MODE 1: up to KIN inputs, dots out·in[j] (j < nin) then out·out (at nin)
// MODE 2: up to KIN inputs (no out), dots in0·in[j] (j < nin) then in1·in[j] (1 <= j < nin)
// KIN is the input capacity the instance is compiled for (the host picks the smallest that
// holds nin): every input and accumulator lives in registers, so capacity costs occupancy --
// a 20-input instance needs 191 registers (one CTA per SM), a 2-input one 40.
#ifndef LC_MINB17
#define LC_MINB17 0         // resident CTAs per SM of the 12- and 17-input instances (0: the compiler's choice)
#endif
template <int MODE, int KIN = (MODE == 0 ? 7 : CL_MAXIN)>
__global__ void __launch_bounds__(NT, (KIN == 17 || KIN == 12) ? LC_MINB17 : 0) lincomb_kernel(LcDev a, int64_t n2, int tail, double* ws,
                                                     double* dots_out) {
    constexpr int ND = MODE == 0 ? 8 : (MODE == 1 ? KIN + 1 : 2 * KIN - 1);
    double acc[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) acc[d] = 0.0;
    const int nin = a.nin;
    const int64_t stride = (int64_t)gridDim.x * NT;
    // element loop over double2 units; the odd tail element is handled by
    // the first thread with a scalar pass folded into the same accumulators
    for (int64_t k = (int64_t)blockIdx.x * NT + threadIdx.x; k < n2 + (tail ? 1 : 0); k += stride) {
        const bool is_tail = (k == n2);
        double2 v[KIN + 1];
#pragma unroll
        for (int j = 0; j < KIN; ++j) {
            if (j < nin) {
                if (!is_tail) v[j] = ld2cs(a.in[j] + 2 * k);
                else v[j] = make_double2(a.in[j][2 * k], 0.0);
            } else {
                v[j] = make_double2(0.0, 0.0);
            }
        }
        double2 o = make_double2(0.0, 0.0);
        if (a.out != nullptr || MODE != 2) {
#pragma unroll
            for (int j = 0; j < KIN; ++j)
                if (j < nin) o = axpy2(a.coef[j], v[j], o);
            if (a.out != nullptr) {
                if (!is_tail) st2(a.out + 2 * k, o);
                else a.out[2 * k] = o.x;
            }
        }
        v[KIN] = o;
        if (MODE == 0) {
#pragma unroll
            for (int d = 0; d < 8; ++d)
                if (d < a.ndot) {
                    int ia = a.da[d] == CL_OUT ? KIN : a.da[d];
                    int ib = a.db[d] == CL_OUT ? KIN : a.db[d];
                    acc[d] += dot2(select2(v, ia), select2(v, ib));
                }
        } else if (MODE == 1) {
#pragma unroll
            for (int j = 0; j < KIN; ++j)
                if (j < nin) acc[j] += dot2(o, v[j]);
            acc[KIN] += dot2(o, o);
        } else {
#pragma unroll
            for (int j = 0; j < KIN; ++j)
                if (j < nin) acc[j] += dot2(v[0], v[j]);
#pragma unroll
            for (int j = 1; j < KIN; ++j)
                if (j < nin) acc[KIN + j - 1] += dot2(v[1], v[j]);
        }
    }
    if (a.ndot > 0) {
        if (MODE == 1) {
            // out·out sits after the nin input dots: move it there (unused slots hold 0)
            if (nin < KIN) {
#pragma unroll
                for (int j = 0; j < KIN; ++j)
                    if (j == nin) acc[j] = acc[KIN];
            }
            reduce_and_finish<ND>(acc, a.ndot, ws, dots_out);
        } else if (MODE == 2) {
            // fixed output layout: [j] = in0·in_j, [CL_MAXIN + j - 1] = in1·in_j
            reduce_and_finish<ND>(acc, a.ndot, ws, dots_out, KIN, CL_MAXIN - KIN);
        } else {
            reduce_and_finish<ND>(acc, a.ndot, ws, dots_out);
        }
    }
}

// ---------------------------------------------------------------------------
// pattern (CSR over positions) times factor, fused coefficient assembly
// ---------------------------------------------------------------------------

struct PatDev {
    int64_t nrows;
    const int64_t* indptr;
    const int32_t* indices;
    const double* cv;
    double c_coeff;
    const int64_t* at_ptr;
    const int32_t* at_con;
    const double* at_val;
    const double* w1;
    const double* w2;
    const double* w1g;    // row-sharded solve: multipliers of constraints owned elsewhere,
    const double* w2g;    // at_con >= mown reads w?g[at_con - mown]
    int64_t mown;
};

__device__ __forceinline__ double wval(const double* w, const double* wg, int64_t mown, int32_t c) {
    return (wg == nullptr || c < mown) ? __ldg(w + c) : __ldg(wg + (c - mown));
}

struct EpiDev {
    int ny;
    const double* Y[CL_MAXY];
    double ycoef[CL_MAXY];
    int nz;
    const double* Z[CL_MAXY];
    int ndot;
    uint8_t da[8], db[8];
    const double* drow;   // optional per-row coefficient of Y[0] (diagonal term), times dmul[row]
    const double* dmul;
    // diagonal-constraint ADMM epilogues (EPI 2: CG start, EPI 3: step end)
    double rho;
    double* rout;         // EPI 2: initial CG residual
    double* cw;           // EPI 2: C Wf itself (optional; the step end reads it back)
    const double* bvec;   // EPI 3: b
    const double* lam;    // EPI 3: multiplier at the step start
    double* axo;          // EPI 3: A(U V^T)
    double* lamo;         // EPI 3: lam + rho (A(U V^T) - b)
};

__device__ __forceinline__ double slot_coef(const PatDev& P, int64_t s) {
    // same association as linops.py:184-194: data = At@w1 + At@w2 + c*cv
    double data = 0.0;
    if (P.at_ptr != nullptr) {
        const int64_t u0 = __ldg(P.at_ptr + s), u1 = __ldg(P.at_ptr + s + 1);
        if (P.w1 != nullptr) {
            double t = 0.0;
            for (int64_t u = u0; u < u1; ++u) t += __ldg(P.at_val + u) * wval(P.w1, P.w1g, P.mown, __ldg(P.at_con + u));
            data += t;
        }
        if (P.w2 != nullptr) {
            double t = 0.0;
            for (int64_t u = u0; u < u1; ++u) t += __ldg(P.at_val + u) * wval(P.w2, P.w2g, P.mown, __ldg(P.at_con + u));
            data += t;
        }
    }
    if (P.cv != nullptr) data += P.c_coeff * __ldg(P.cv + s);
    return data;
}

// One group of G lanes per row; lane l owns columns {2l, 2l+1} + 2G*c.
// VEC = 1 only for ld == 1 (Lanczos vectors).
template <int G, int VEC>
__global__ void __launch_bounds__(NT) pattern_spmm_kernel(PatDev P, const double* __restrict__ X, int ld,
                                                          double alpha, EpiDev E, double* out,
                                                          double* ws, double* dots_out) {
    constexpr int NOPS = 2 * CL_MAXY + 1;   // Y[0..3], out(4)->index CL_MAXY, Z[0..3] at 5..8
    double acc[8];
#pragma unroll
    for (int d = 0; d < 8; ++d) acc[d] = 0.0;
    const int lane = threadIdx.x & 31;
    const int gl = lane % G;                       // lane within group
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane - gl));
    const int64_t groups_total = (int64_t)gridDim.x * (NT / G);
    const int64_t g0 = ((int64_t)blockIdx.x * NT + threadIdx.x) / G;
    const int ncol_chunk = G * VEC;

    for (int64_t row = g0; row < P.nrows + 0; row += groups_total) {
        const int64_t s0 = __ldg(P.indptr + row), s1 = __ldg(P.indptr + row + 1);
        for (int c0 = 0; c0 < ld; c0 += ncol_chunk) {
            const int col = c0 + gl * VEC;
            const bool active = col < ld;
            double2 sum = make_double2(0.0, 0.0);
            for (int64_t base = s0; base < s1; base += G) {
                const int64_t s = base + gl;
                int jj = 0;
                double cc = 0.0;
                if (s < s1) {
                    jj = __ldg(P.indices + s);
                    cc = slot_coef(P, s);
                }
                const int cnt = (int)min((int64_t)G, s1 - base);
#pragma unroll 4
                for (int t = 0; t < cnt; ++t) {
                    const int j = __shfl_sync(gmask, jj, (lane - gl) + t);
                    const double c = __shfl_sync(gmask, cc, (lane - gl) + t);
                    if (active) {
                        if (VEC == 2) {
                            double2 x = ld2(X + (int64_t)j * ld + col);
                            sum.x = fma(c, x.x, sum.x);
                            sum.y = fma(c, x.y, sum.y);
                        } else {
                            sum.x = fma(c, __ldg(X + (int64_t)j * ld + col), sum.x);
                        }
                    }
                }
            }
            if (active) {
                const int64_t off = row * (int64_t)ld + col;
                double2 ops[NOPS];
                double2 o = make_double2(alpha * sum.x, alpha * sum.y);
#pragma unroll
                for (int j = 0; j < CL_MAXY; ++j) {
                    if (j < E.ny) {
                        double2 y = VEC == 2 ? ld2cs(E.Y[j] + off) : make_double2(E.Y[j][off], 0.0);
                        ops[j] = y;
                        o = axpy2(E.ycoef[j], y, o);
                    } else {
                        ops[j] = make_double2(0.0, 0.0);
                    }
                }
                if (VEC == 1) o.y = 0.0;
                ops[CL_MAXY] = o;
#pragma unroll
                for (int j = 0; j < CL_MAXY; ++j) {
                    if (j < E.nz) ops[CL_MAXY + 1 + j] = VEC == 2 ? ld2cs(E.Z[j] + off) : make_double2(E.Z[j][off], 0.0);
                    else ops[CL_MAXY + 1 + j] = make_double2(0.0, 0.0);
                }
                if (out != nullptr) {
                    if (VEC == 2) st2(out + off, o);
                    else out[off] = o.x;
                }
#pragma unroll
                for (int d = 0; d < 8; ++d)
                    if (d < E.ndot) {
                        int ia = E.da[d] == CL_OUT ? CL_MAXY : (E.da[d] >= 16 ? CL_MAXY + 1 + (E.da[d] - 16) : E.da[d]);
                        int ib = E.db[d] == CL_OUT ? CL_MAXY : (E.db[d] >= 16 ? CL_MAXY + 1 + (E.db[d] - 16) : E.db[d]);
                        acc[d] += dot2(select2(ops, ia), select2(ops, ib));
                    }
            }
        }
    }
    if (E.ndot > 0) reduce_and_finish<8>(acc, E.ndot, ws, dots_out);
}

// ---------------------------------------------------------------------------
// fused A(X Y^T): compressed outer product + stacked constraint product
// ---------------------------------------------------------------------------

template <int G, int VEC>
__device__ __forceinline__ double group_dot(const double* __restrict__ X, const double* __restrict__ Y,
                                            int64_t i, int64_t j, int ld, int gl, unsigned gmask) {
    double p = 0.0;
    for (int col = gl * VEC; col < ld; col += G * VEC) {
        if (VEC == 2) p += dot2(ld2(X + i * ld + col), ld2(Y + j * ld + col));
        else p += __ldg(X + i * ld + col) * __ldg(Y + j * ld + col);
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) p += __shfl_xor_sync(gmask, p, o);
    return p;
}

// Ghost rows of the row-sharded solve for the six operands of constraint_kernel
// (row index >= nown reads g[k][row - nown]); nown < 0: no ghost rows.
struct ConGhost {
    const double* g[6];
    int64_t nown;
    int64_t sx;           // row stride of the local operands (ld; 2 ld for a pair buffer)
};

// nown == CL_GHOST_PEERS: position index i < 0 is CL_PEER_COL(owner, row), read in place
// from operand k's row block on the owner rank, p[k][owner] (include/culorads.h)
struct ConPeers {
    const double* p[6][CL_MAX_PEERS];
};

__device__ __forceinline__ const double* grow(const double* X, const double* Xg, int64_t i, int64_t nown, int ld,
                                              int64_t sx) {
    return (nown < 0 || i < nown) ? X + i * sx : Xg + (i - nown) * ld;
}

// Row i of constraint operand k: local, halo buffer (i >= nown), or (PEER) a peer's memory.
#define growk(PEER, X, gh, k, i, nown, ld)                                                                  \
    ((PEER) && (i) < 0 ? pp.p[k][((uint32_t)(i) >> CL_PEER_ROW_BITS) & (CL_MAX_PEERS - 1)] +                  \
                             (int64_t)((uint32_t)(i) & CL_PEER_ROW_MASK) * (gh).sx                             \
                       : grow(X, (gh).g[k], i, nown, ld, (gh).sx))

template <int G, int VEC>
__device__ __forceinline__ double group_dot_rows(const double* __restrict__ x, const double* __restrict__ y, int ld,
                                                 int gl, unsigned gmask) {
    double p = 0.0;
    for (int col = gl * VEC; col < ld; col += G * VEC) {
        if (VEC == 2) p += dot2(ld2(x + col), ld2(y + col));
        else p += __ldg(x + col) * __ldg(y + col);
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) p += __shfl_xor_sync(gmask, p, o);
    return p;
}

// Resident CTAs per SM the constraint kernel (A(UV^T)) and the single-entry ADMM operator
// are compiled for (a register cap). Unset: the compiler's own choice -- note that an
// explicit minBlocks of 1 is NOT the same (it lets ptxas spend up to 86 registers).
#ifndef CK_MINB
#define CK_MINB 6           // A(UV^T): 40 registers, 6 CTAs/SM: 5.77 -> 4.49 ms at configs[3]'s share
#endif
#ifndef CK3_MINB
#define CK3_MINB 0          // the line search's three-product variant: the compiler's choice
#endif
#define CK_BOUNDS(NP) __launch_bounds__(NT, (NP) == 1 ? CK_MINB : CK3_MINB)   // 0: the compiler's choice
#ifndef SE_U
#define SE_U 2              // slots whose row gathers the single-entry operator issues together (1: 6.20 ms, 2: 5.62, 4: 6.54 at configs[3]'s share)
#endif
#ifdef SE_MINB
#define SE_BOUNDS __launch_bounds__(NT, SE_MINB)
#else
#define SE_BOUNDS __launch_bounds__(NT)
#endif

template <int G, int VEC, int NP, int PEER = 0>    // NP = 1: X1 Y1 only (A(UV^T)); 3: up to three products
__global__ void CK_BOUNDS(NP) constraint_kernel(int64_t m, const int64_t* __restrict__ indptr,
                                                        const int32_t* __restrict__ pi,
                                                        const int32_t* __restrict__ pj,
                                                        const double* __restrict__ val, int ld,
                                                        const double* X1, const double* Y1,
                                                        const double* X2, const double* Y2, double* out1,
                                                        const double* X3, const double* Y3, double* out2,
                                                        ConGhost gh, ConPeers pp) {
    const int lane = threadIdx.x & 31;
    const int gl = lane % G;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane - gl));
    const int64_t groups_total = (int64_t)gridDim.x * (NT / G);
    const int64_t nw = gh.nown;
    if (VEC == 2 && ld <= 2 * G) {
        // One double2 per lane per row: the positions of two nonzeros are read, then all
        // their gathers are issued together, then reduced in the order of the general
        // loop below (same arithmetic, bit for bit; fewer dependent memory round trips).
        const int col = gl * 2;
        const bool act = col < ld;
        const double2 z2 = make_double2(0.0, 0.0);
        for (int64_t c = ((int64_t)blockIdx.x * NT + threadIdx.x) / G; c < m; c += groups_total) {
            const int64_t t0 = __ldg(indptr + c), t1 = __ldg(indptr + c + 1);
            double a1 = 0.0, a2 = 0.0;
            for (int64_t t = t0; t < t1; t += 2) {
                const bool two = t + 1 < t1;
                const int64_t i0 = __ldg(pi + t), j0 = __ldg(pj + t);
                const int64_t i1 = two ? (int64_t)__ldg(pi + t + 1) : i0, j1 = two ? (int64_t)__ldg(pj + t + 1) : j0;
                const double v0 = __ldg(val + t), v1 = two ? __ldg(val + t + 1) : 0.0;
                double2 x1a = z2, y1a = z2, x1b = z2, y1b = z2, x2a = z2, y2a = z2, x2b = z2, y2b = z2;
                double2 x3a = z2, y3a = z2, x3b = z2, y3b = z2;
                if (act) {
                    x1a = ld2(growk(PEER, X1, gh, 0, i0, nw, ld) + col);
                    y1a = ld2(growk(PEER, Y1, gh, 1, j0, nw, ld) + col);
                    if (two) {
                        x1b = ld2(growk(PEER, X1, gh, 0, i1, nw, ld) + col);
                        y1b = ld2(growk(PEER, Y1, gh, 1, j1, nw, ld) + col);
                    }
                    if (NP > 1 && X2 != nullptr) {
                        x2a = ld2(growk(PEER, X2, gh, 2, i0, nw, ld) + col);
                        y2a = ld2(growk(PEER, Y2, gh, 3, j0, nw, ld) + col);
                        if (two) {
                            x2b = ld2(growk(PEER, X2, gh, 2, i1, nw, ld) + col);
                            y2b = ld2(growk(PEER, Y2, gh, 3, j1, nw, ld) + col);
                        }
                    }
                    if (NP > 1 && X3 != nullptr) {
                        x3a = ld2(growk(PEER, X3, gh, 4, i0, nw, ld) + col);
                        y3a = ld2(growk(PEER, Y3, gh, 5, j0, nw, ld) + col);
                        if (two) {
                            x3b = ld2(growk(PEER, X3, gh, 4, i1, nw, ld) + col);
                            y3b = ld2(growk(PEER, Y3, gh, 5, j1, nw, ld) + col);
                        }
                    }
                }
                double p1a = 0.0, p1b = 0.0, p2a = 0.0, p2b = 0.0, p3a = 0.0, p3b = 0.0;
                if (act) {
                    p1a += dot2(x1a, y1a);
                    p1b += dot2(x1b, y1b);
                    if (NP > 1) {
                        p2a += dot2(x2a, y2a);
                        p2b += dot2(x2b, y2b);
                        p3a += dot2(x3a, y3a);
                        p3b += dot2(x3b, y3b);
                    }
                }
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) {
                    p1a += __shfl_xor_sync(gmask, p1a, o);
                    p1b += __shfl_xor_sync(gmask, p1b, o);
                    if (NP > 1) {
                        p2a += __shfl_xor_sync(gmask, p2a, o);
                        p2b += __shfl_xor_sync(gmask, p2b, o);
                        p3a += __shfl_xor_sync(gmask, p3a, o);
                        p3b += __shfl_xor_sync(gmask, p3b, o);
                    }
                }
                double xa = p1a, xb = p1b;
                if (NP > 1 && X2 != nullptr) {
                    xa += p2a;
                    xb += p2b;
                }
                a1 += v0 * xa;
                if (NP > 1 && X3 != nullptr) a2 += v0 * p3a;
                if (two) {
                    a1 += v1 * xb;
                    if (NP > 1 && X3 != nullptr) a2 += v1 * p3b;
                }
            }
            if (gl == 0) {
                out1[c] = a1;
                if (X3 != nullptr) out2[c] = a2;
            }
        }
        return;
    }
    for (int64_t c = ((int64_t)blockIdx.x * NT + threadIdx.x) / G; c < m; c += groups_total) {
        const int64_t t0 = __ldg(indptr + c), t1 = __ldg(indptr + c + 1);
        double a1 = 0.0, a2 = 0.0;
        for (int64_t t = t0; t < t1; ++t) {
            const int64_t i = __ldg(pi + t), j = __ldg(pj + t);
            const double v = __ldg(val + t);
            double x = group_dot_rows<G, VEC>(growk(PEER, X1, gh, 0, i, nw, ld), growk(PEER, Y1, gh, 1, j, nw, ld), ld, gl,
                                              gmask);
            if (X2 != nullptr)
                x += group_dot_rows<G, VEC>(growk(PEER, X2, gh, 2, i, nw, ld), growk(PEER, Y2, gh, 3, j, nw, ld), ld, gl,
                                            gmask);
            a1 += v * x;
            if (X3 != nullptr)
                a2 += v * group_dot_rows<G, VEC>(growk(PEER, X3, gh, 4, i, nw, ld), growk(PEER, Y3, gh, 5, j, nw, ld), ld, gl,
                                                 gmask);
        }
        if (gl == 0) {
            out1[c] = a1;
            if (X3 != nullptr) out2[c] = a2;
        }
    }
}

template <int G, int VEC>
__global__ void __launch_bounds__(NT) sddmm_kernel(int64_t K, const int32_t* __restrict__ imap,
                                                   const int32_t* __restrict__ jmap, int ld,
                                                   const double* X, const double* Y, double* x) {
    const int lane = threadIdx.x & 31;
    const int gl = lane % G;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane - gl));
    const int64_t groups_total = (int64_t)gridDim.x * (NT / G);
    for (int64_t k = ((int64_t)blockIdx.x * NT + threadIdx.x) / G; k < K; k += groups_total) {
        double p = group_dot<G, VEC>(X, Y, __ldg(imap + k), __ldg(jmap + k), ld, gl, gmask);
        if (gl == 0) x[k] = p;
    }
}

// Diagonal constraints (constraint c is a_c e_c e_c^T, MaxCut): the stacked
// product collapses to row dot products, streamed with no index traffic.
// The host resolves operand aliasing (the line search passes R and D in six
// roles) into <= 6 distinct streams; each group loads the distinct rows of DR
// rows in one batch, then reduces every product exactly like group_dot, so
// results equal constraint_kernel's bit for bit.
struct DiagCon {
    int64_t n;
    const double* aval;
    int ld;
    int nop;                  // distinct operand streams
    const double* op[6];
    int pidx[6];              // (x, y) stream of product 1, 2, 3
    int nprod1;               // products summed into out1 (1 or 2)
    double* out1;
    double* out2;             // product 3 (NULL: none)
};

template <int VEC>
__device__ __forceinline__ double2 ldrow(const double* p, int64_t off) {
    return VEC == 2 ? ld2(p + off) : make_double2(__ldg(p + off), 0.0);
}

template <int G, int VEC, int NOP>
__global__ void __launch_bounds__(NT, 4) diag_constraint_kernel(DiagCon a) {
    constexpr int DR = NOP <= 2 ? 2 : 1;
    const int lane = threadIdx.x & 31;
    const int gl = lane % G;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane - gl));
    const int64_t gt = (int64_t)gridDim.x * (NT / G);
    const bool two = a.nprod1 == 2, three = a.out2 != nullptr;
    const int ld = a.ld;
    for (int64_t cb = ((int64_t)blockIdx.x * NT + threadIdx.x) / G; cb < a.n; cb += DR * gt) {
        double p[DR][3];
#pragma unroll
        for (int u = 0; u < DR; ++u) p[u][0] = p[u][1] = p[u][2] = 0.0;
        for (int col = gl * VEC; col < ld; col += G * VEC) {
            double2 v[DR][NOP];
#pragma unroll
            for (int u = 0; u < DR; ++u) {
                const int64_t c = cb + u * gt;
                const int64_t off = c * ld + col;
#pragma unroll
                for (int k = 0; k < NOP; ++k)
                    v[u][k] = (k < a.nop && c < a.n) ? ldrow<VEC>(a.op[k], off) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < DR; ++u) {
                p[u][0] += dot2(select2(v[u], a.pidx[0]), select2(v[u], a.pidx[1]));
                if (two) p[u][1] += dot2(select2(v[u], a.pidx[2]), select2(v[u], a.pidx[3]));
                if (three) p[u][2] += dot2(select2(v[u], a.pidx[4]), select2(v[u], a.pidx[5]));
            }
        }
#pragma unroll
        for (int u = 0; u < DR; ++u) {
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) {
                p[u][0] += __shfl_xor_sync(gmask, p[u][0], o);
                if (two) p[u][1] += __shfl_xor_sync(gmask, p[u][1], o);
                if (three) p[u][2] += __shfl_xor_sync(gmask, p[u][2], o);
            }
            const int64_t c = cb + u * gt;
            if (gl == 0 && c < a.n) {
                const double w = __ldg(a.aval + c);
                const double x = two ? p[u][0] + p[u][1] : p[u][0];
                a.out1[c] = 0.0 + w * x;
                if (three) a.out2[c] = 0.0 + w * p[u][2];
            }
        }
    }
}

// Flat variant for even ld: a block streams RB whole rows as one contiguous
// run of double2 units (every warp load is 512 contiguous bytes, U loads in
// flight per thread), parks the per-unit products in shared memory and lets
// one thread per row fold its units in order. Products 1 and 2 are summed
// per unit (q1 = A(R D^T + D R^T) in the line search).
#ifndef DC_U
#define DC_U 4              // units in flight per thread of the flat row kernels: A(RR^T) 0.49 -> 0.35 ms, CG apply 2.06 -> 1.47 ms at n = 1e7 (8 was register-bound)
#endif
#ifndef CL_SMALLN
#define CL_SMALLN 1         // small problems: spread rows over at least FLAT_MIN_BLK blocks / one tile per CTA
#endif
#define FLAT_MIN_BLK (2 * NSM)
#ifndef DCF_MAXH2
#define DCF_MAXH2 32        // widest row (double2 units) the flat diagonal-constraint kernel takes
#endif

// Rows per block iteration of the flat row kernels: NT*DC_U double2 units, or fewer when
// that would leave SMs idle (small n), so every SM has work and each thread few units.
__host__ __device__ __forceinline__ int flat_rows(int64_t n, int h2) {
    int rb = (NT * DC_U) / h2;
#if CL_SMALLN
    const int64_t spread = (n + FLAT_MIN_BLK - 1) / FLAT_MIN_BLK;
    if (spread < rb) rb = spread < 1 ? 1 : (int)spread;
#endif
    return rb;
}

template <int NOP>
__global__ void __launch_bounds__(NT) diag_constraint_flat_kernel(DiagCon a) {
    __shared__ double part[2][NT * DC_U];
    const int h2 = a.ld >> 1;
    const int rb = flat_rows(a.n, h2);                // rows per block iteration (>= 1)
    const bool two = a.nprod1 == 2, three = a.out2 != nullptr;
    const int64_t nblk = (a.n + rb - 1) / rb;
    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const int64_t r0 = blk * rb;
        const int nr = (int)min((int64_t)rb, a.n - r0);
        const int units = nr * h2;
        const int64_t base = r0 * (int64_t)h2;         // first double2 unit
        double2 v[DC_U][NOP];
#pragma unroll
        for (int u = 0; u < DC_U; ++u) {
            const int e = threadIdx.x + u * NT;
#pragma unroll
            for (int k = 0; k < NOP; ++k)
                v[u][k] = (e < units && k < a.nop) ? ld2(a.op[k] + 2 * (base + e)) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < DC_U; ++u) {
            const int e = threadIdx.x + u * NT;
            if (e < units) {
                double x = dot2(select2(v[u], a.pidx[0]), select2(v[u], a.pidx[1]));
                if (two) x += dot2(select2(v[u], a.pidx[2]), select2(v[u], a.pidx[3]));
                part[0][e] = x;
                if (three) part[1][e] = dot2(select2(v[u], a.pidx[4]), select2(v[u], a.pidx[5]));
            }
        }
        __syncthreads();
        for (int r = threadIdx.x; r < nr; r += NT) {
            double s1 = 0.0, s3 = 0.0;
            for (int q = 0; q < h2; ++q) {
                s1 += part[0][r * h2 + q];
                if (three) s3 += part[1][r * h2 + q];
            }
            const double w = __ldg(a.aval + r0 + r);
            a.out1[r0 + r] = w * s1;
            if (three) a.out2[r0 + r] = w * s3;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// diagonal-constraint (MaxCut-shaped) fused ALM update
// ---------------------------------------------------------------------------

struct DiagDev {
    int64_t n;
    int ld;
    const double* aval;
    double tau, rho, scale;
    double* R; const double* D; double* CR; const double* CD;
    const double* ax; double* ax_out; const double* q1; const double* q2;
    const double* lam; const double* b;
    const double* g_old; double* g_new; double* y;
    int nh;
    const double* H[CL_MAXIN];
    int refresh;
};

// Dots (fixed layout, see culorads.h):
//  0 <CR,R>  1 <g,g>  2 <y,D>  3 lam·res  4 res·res  5 <y,y>  6 <g,y>
//  7+h <g,H_h>   7+CL_MAXIN+h <y,H_h>
// One thread per double2 of the flat n*ld factor; every thread of a row
// recomputes the row's constraint scalars from the (read-only) m-vectors and
// the row owner (first double2 of the row) writes ax_out and adds the m-dots.
#ifndef DU_DIV32
#define DU_DIV32 1
#endif
#ifndef DU_B17
#define DU_B17 1            // a history bucket of exactly 17 (2 * memory + 1 at memory 8): 12.2 -> 9.6 ms at n = 1e7
#endif
#ifndef DU_MINB
#define DU_MINB 3           // resident CTAs per SM of the 4- and 10-wide buckets (10: 7.6 -> 6.5 ms at n = 1e7)
#endif
// (tools/diag_update_probe.py, profiles/r2_final/diag_update_probe.jsonl; the wider buckets
// are fastest at the compiler's own register choice)
template <int NH, bool GOLD = true>   // GOLD false: g_old = 0 (the inner solve's first gradient)
__global__ void __launch_bounds__(NT, (NH == 4 || NH == 10) ? DU_MINB : 0) diag_update_kernel(DiagDev a, double* ws, double* dots_out) {
    constexpr int ND = 7 + 2 * NH;
    double acc[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) acc[d] = 0.0;
    const int half = a.ld >> 1;
    const int64_t n2 = a.n * half;
    const int64_t stride = (int64_t)gridDim.x * NT;
    // 32-bit row division (the 64-bit one is a long call) in the history buckets: the 10-wide
    // one gains 6 % at n = 1e7; the history-free instance, whose refresh pass is the bench's
    // gradient, measured faster with the 64-bit one (1.89 against 2.06 ms; code generation,
    // not the division itself -- profiles/r2_final/diag_update_probe.jsonl)
    constexpr bool DIV32 = DU_DIV32 && NH > 0;
    const bool small = n2 < (int64_t(1) << 32);
    for (int64_t k = (int64_t)blockIdx.x * NT + threadIdx.x; k < n2; k += stride) {
        const int64_t row = DIV32 && small ? (int64_t)((uint32_t)k / (uint32_t)half) : k / half;
        const bool owner = (k - row * half) == 0;
        double axr = __ldg(a.ax + row);
        if (!a.refresh) axr = axr + a.tau * __ldg(a.q1 + row) + a.tau * a.tau * __ldg(a.q2 + row);
        const double res = axr - __ldg(a.b + row);
        const double lam = __ldg(a.lam + row);
        const double w = lam + a.rho * res;
        if (owner) {
            a.ax_out[row] = axr;
            acc[3] += lam * res;
            acc[4] += res * res;
        }
        const double wa = w * __ldg(a.aval + row);
        const int64_t off = 2 * k;
        double2 R = ld2cs(a.R + off), CR = ld2cs(a.CR + off);
        const double2 D = ld2cs(a.D + off);
        if (!a.refresh) {
            const double2 CD = ld2cs(a.CD + off);
            R = axpy2(a.tau, D, R);
            CR = axpy2(a.tau, CD, CR);
            st2(a.R + off, R);
            st2(a.CR + off, CR);
        }
        // g = 2 S R with S = scale*C + A*(w): 2*(w_i a_i R_i + scale*CR_i)  (alm.py:245)
        double2 g;
        g.x = 2.0 * (wa * R.x + a.scale * CR.x);
        g.y = 2.0 * (wa * R.y + a.scale * CR.y);
        const double2 go = GOLD ? ld2cs(a.g_old + off) : make_double2(0.0, 0.0);
        const double2 y = make_double2(g.x - go.x, g.y - go.y);
        st2(a.g_new + off, g);
        st2(a.y + off, y);
        acc[0] += dot2(CR, R);
        acc[1] += dot2(g, g);
        acc[2] += dot2(y, D);
        acc[5] += dot2(y, y);
        acc[6] += dot2(g, y);
#pragma unroll
        for (int h = 0; h < NH; ++h)
            if (h < a.nh) {
                const double2 hv = ld2cs(a.H[h] + off);
                acc[7 + h] += dot2(g, hv);
                acc[7 + NH + h] += dot2(y, hv);
            }
    }
    // dots_out layout is fixed by the ABI (7 + 2*CL_MAXIN): the y-row lands at 7 + CL_MAXIN
    reduce_and_finish<ND>(acc, ND, ws, dots_out, 7 + NH, CL_MAXIN - NH);
}

// ---------------------------------------------------------------------------
// Lanczos basis projections
// ---------------------------------------------------------------------------

#define BP_TILE 8
#define BP_CHUNKS NSM

__global__ void __launch_bounds__(NT) basis_project_kernel(const double* __restrict__ Q, int64_t ldq, int kc,
                                                           int64_t n, const double* __restrict__ v,
                                                           double* ws) {
    const int chunk = blockIdx.x;
    const int t0 = blockIdx.y * BP_TILE;
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t k0 = chunk * per, k1 = min(n, k0 + per);
    double acc[BP_TILE];
#pragma unroll
    for (int t = 0; t < BP_TILE; ++t) acc[t] = 0.0;
    for (int64_t k = k0 + threadIdx.x; k < k1; k += NT) {
        const double vk = __ldg(v + k);
#pragma unroll
        for (int t = 0; t < BP_TILE; ++t)
            if (t0 + t < kc) acc[t] += __ldg(Q + (int64_t)(t0 + t) * ldq + k) * vk;
    }
    __shared__ double sh[NWARP][BP_TILE];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int t = 0; t < BP_TILE; ++t) {
        double s = warp_sum(acc[t]);
        if (lane == 0) sh[wid][t] = s;
    }
    __syncthreads();
    if (threadIdx.x < BP_TILE && t0 + threadIdx.x < kc) {
        double s = 0.0;
        for (int w = 0; w < NWARP; ++w) s += sh[w][threadIdx.x];
        ws[(int64_t)chunk * kc + t0 + threadIdx.x] = s;
    }
}

// h[t] = sum over chunks of the partials: a warp per t (lanes stride over the chunks, a
// shuffle tree), so the chunk loads are in flight together -- one thread per t read them
// one after another and cost 26 us per Gram-Schmidt pass at n = 2e5
__global__ void basis_project_finish(const double* ws, int nchunks, int kc, double* h) {
    const int lane = threadIdx.x & 31;
    const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (t >= kc) return;
    double s = 0.0;
    for (int c = lane; c < nchunks; c += 32) s += ws[(int64_t)c * kc + t];
    s = warp_sum(s);
    if (lane == 0) h[t] = s;
}

__global__ void __launch_bounds__(NT) basis_subtract_kernel(const double* __restrict__ Q, int64_t ldq, int kc,
                                                            int64_t n, const double* __restrict__ h,
                                                            double* v) {
    extern __shared__ double hs[];
    for (int t = threadIdx.x; t < kc; t += NT) hs[t] = h[t];
    __syncthreads();
    for (int64_t k = (int64_t)blockIdx.x * NT + threadIdx.x; k < n; k += (int64_t)gridDim.x * NT) {
        double s = 0.0;
        for (int t = 0; t < kc; ++t) s += hs[t] * __ldg(Q + (int64_t)t * ldq + k);
        v[k] -= s;
    }
}

// ---------------------------------------------------------------------------
// tiled CSR SpMM: row segments staged in shared memory by the bulk-copy
// (TMA) engine, one tile ahead, so the factor-row gathers are the only
// global loads on the critical path (linops.py:122 spmm)
// ---------------------------------------------------------------------------

#ifndef SP_SMAX
#define SP_SMAX 1024        // slots staged per tile (indices + values)
#endif
#define SP_PTRMAX 264       // row pointers per tile: TR + 1 + alignment slack, TR <= 256
#ifndef SP_UNROLL
#define SP_UNROLL 5         // gathers in flight per lane (epilogue variants): 4 % faster than 4, 12-17 % than 8 (profiles/r2_peer)
#endif
// Plain-store variant: more gathers in flight for narrow rows (12: 4.32 -> 4.12 ms for C R at
// n = 1e7, ld 26), fewer for wide rows where one group already covers 512 bytes per gather
// (4: 13.3 -> 12.6 ms at ld 822); the epilogue variants lose registers to more (occupancy_sweep).
#ifndef SP_UNROLL0
#define SP_UNROLL0 10        // plain store, narrow rows: 4.15 ms against 4.38 ms at 12 (n = 1e7, ld 26; profiles/r2_peer)
#endif
#ifndef SP_UNROLL0_WIDE
#define SP_UNROLL0_WIDE 4
#endif
#ifndef SP_MINB2
#define SP_MINB2 3          // the diagonal ADMM epilogues (CG start, step end)
#endif
#ifndef SP_UNROLLG
#define SP_UNROLLG 6        // gathers in flight per lane, plain store with ghost rows (12 spills at 64 registers)
#endif
#ifndef SP_UNROLLGE
#define SP_UNROLLGE 4       // the same for the epilogue variants with ghost rows
#endif
#ifndef SP_MINBGE
#define SP_MINBGE 4         // resident CTAs per SM of the epilogue variants with ghost rows
#endif
#ifndef SP_UNROLL2
#define SP_UNROLL2 SP_UNROLL  // gathers in flight per lane, diagonal-ADMM epilogues
#endif
#ifndef SP_MINBG
#define SP_MINBG 4          // plain-store variants with ghost rows (halo buffer / peer memory)
#endif
#ifndef SP_MINB1
#define SP_MINB1 3          // resident CTAs per SM the epilogue variants are compiled for
#endif
#ifndef SP_MINB0
#define SP_MINB0 4          // resident CTAs per SM the plain-epilogue variant is compiled for
#endif
#define SP_NY 2             // epilogue limits of the tiled path (else the row-group kernel)
#define SP_NZ 3
#define SP_ND 4

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

struct SpDev {
    int64_t nrows;
    const int64_t* indptr;
    const int32_t* indices;
    const double* vals;
    const double* X;
    const double* Xg;     // ghost rows (row-sharded solve): column j >= nown reads Xg[j - nown]
    int32_t nown;         // INT32_MAX when there is no ghost block
    // peer-memory ghosts (GHOST 2): a remote column is encoded as CL_PEER_COL(owner, row)
    // and read in place from the owner's factor, Xp[owner] + row * ld (NVLink loads)
    const double* Xp[CL_MAX_PEERS];
    int ld;
    double alpha;
    double* out;
    int tr;               // rows per tile (multiple of the group count)
    int64_t ntiles;
};

struct SpTile {
    int64_t ptr[SP_PTRMAX];
    int32_t idx[SP_SMAX + 8];
    double val[SP_SMAX + 4];
};

// Thread 0: stage tile `tile` (slot range [s0, s1)) into buffer `buf`.
// Sources are read as 16-byte aligned supersets (the host pads every array).
__device__ __forceinline__ void sp_issue(const SpDev& a, SpTile* T, int64_t (*meta)[4], uint64_t* bar, int buf,
                                         int64_t tile, int64_t s0, int64_t s1) {
    const int64_t r0 = tile * a.tr;
    const int64_t r1 = min(r0 + (int64_t)a.tr, a.nrows);
    const int64_t pb = r0 & ~1LL, pe = (r1 + 2) & ~1LL;
    const bool heavy = (s1 - s0) > SP_SMAX;
    const int64_t ib = s0 & ~3LL, ie = (s1 + 3) & ~3LL;
    const int64_t vb = s0 & ~1LL, ve = (s1 + 1) & ~1LL;
    const uint32_t pbytes = (uint32_t)((pe - pb) * 8);
    const uint32_t ibytes = heavy ? 0u : (uint32_t)((ie - ib) * 4);
    const uint32_t vbytes = heavy ? 0u : (uint32_t)((ve - vb) * 8);
    meta[buf][0] = pb;
    meta[buf][1] = ib;
    meta[buf][2] = vb;
    meta[buf][3] = heavy ? 1 : 0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_tx(&bar[buf], pbytes + ibytes + vbytes);
    bulk_g2s(T[buf].ptr, a.indptr + pb, pbytes, &bar[buf]);
    if (ibytes) bulk_g2s(T[buf].idx, a.indices + ib, ibytes, &bar[buf]);
    if (vbytes) bulk_g2s(T[buf].val, a.vals + vb, vbytes, &bar[buf]);
}

// Source row of pattern column j: own rows from X; GHOST 1: rows >= nown from the halo
// buffer; GHOST 2: negative (encoded) columns straight from the owner rank's memory.
template <int GHOST>
__device__ __forceinline__ const double* sp_src(const SpDev& a, const double* X, int j, int ld) {
    if (GHOST == 1 && j >= a.nown) return a.Xg + (int64_t)(j - a.nown) * ld;
    if (GHOST == 2 && j < 0) {
        const uint32_t u = (uint32_t)j;
        return a.Xp[(u >> CL_PEER_ROW_BITS) & (CL_MAX_PEERS - 1)] + (int64_t)(u & CL_PEER_ROW_MASK) * ld;
    }
    return X + (int64_t)j * ld;
}

template <int G, int VEC, int EPI, int GHOST>
__global__ void __launch_bounds__(NT, EPI == 0 ? (GHOST ? SP_MINBG : SP_MINB0) : (GHOST ? SP_MINBGE : (EPI >= 2 ? SP_MINB2 : SP_MINB1))) spmm_tiled_kernel(SpDev a, EpiDev E, double* ws,
                                                                                     double* dots_out) {
    constexpr int NG = NT / G;
    constexpr int SPU = EPI == 0 ? (G == 32 ? SP_UNROLL0_WIDE : (GHOST ? SP_UNROLLG : SP_UNROLL0))
                                 : (GHOST ? SP_UNROLLGE : (EPI >= 2 ? SP_UNROLL2 : SP_UNROLL));
    // epilogue operand set of the tiled path: Y0, Y1, out, Z0, Z1, Z2
    constexpr int NOPS = SP_NY + 1 + SP_NZ;
    __shared__ __align__(128) SpTile T[2];
    __shared__ int64_t meta[2][4];
    __shared__ __align__(8) uint64_t bar[2];
    double dacc[SP_ND];
#pragma unroll
    for (int d = 0; d < SP_ND; ++d) dacc[d] = 0.0;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int gl = lane % G;
    const int grp = tid / G;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane - gl));
    const int rpg = a.tr / NG;
    const int ld = a.ld;
    const double* __restrict__ X = a.X;

    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    int64_t t = blockIdx.x;
    const int64_t stride = gridDim.x;
    int64_t nx0 = 0, nx1 = 0;        // slot bounds of tile t + stride (thread 0)
    if (tid == 0 && t < a.ntiles) {
        const int64_t r0 = t * a.tr, r1 = min(r0 + (int64_t)a.tr, a.nrows);
        sp_issue(a, T, meta, bar, 0, t, __ldg(a.indptr + r0), __ldg(a.indptr + r1));
        if (t + stride < a.ntiles) {
            const int64_t q0 = (t + stride) * a.tr, q1 = min(q0 + (int64_t)a.tr, a.nrows);
            nx0 = __ldg(a.indptr + q0);
            nx1 = __ldg(a.indptr + q1);
        }
    }
    uint32_t phase = 0;   // bit b: parity of buffer b's next completion
    int buf = 0;
    for (; t < a.ntiles; t += stride, buf ^= 1) {
        if (tid == 0) {
            const int64_t tn = t + stride;
            if (tn < a.ntiles) {
                sp_issue(a, T, meta, bar, buf ^ 1, tn, nx0, nx1);
                const int64_t tnn = tn + stride;
                if (tnn < a.ntiles) {
                    const int64_t q0 = tnn * a.tr, q1 = min(q0 + (int64_t)a.tr, a.nrows);
                    nx0 = __ldg(a.indptr + q0);
                    nx1 = __ldg(a.indptr + q1);
                }
            }
        }
        mbar_wait(&bar[buf], (phase >> buf) & 1u);
        phase ^= (1u << buf);
        const SpTile& B = T[buf];
        const int64_t pb = meta[buf][0], ib = meta[buf][1], vb = meta[buf][2];
        const bool heavy = meta[buf][3] != 0;
        const int64_t r0 = t * a.tr;
        const int64_t nr = min((int64_t)a.tr, a.nrows - r0);
        for (int k = 0; k < rpg; ++k) {
            const int lr = grp * rpg + k;
            if (lr >= nr) break;
            const int64_t row = r0 + lr;
            const int64_t s0 = B.ptr[row - pb], s1 = B.ptr[row + 1 - pb];
            double pd_row = 0.0;     // EPI 2/3: the row dot <Z0_i, Y0_i> over all column chunks
            if (EPI >= 2) {
                for (int c = gl * VEC; c < ld; c += G * VEC)
                    pd_row += dot2(ld2cs(E.Z[0] + row * (int64_t)ld + c), ld2cs(E.Y[0] + row * (int64_t)ld + c));
#pragma unroll
                for (int sh = G / 2; sh > 0; sh >>= 1) pd_row += __shfl_xor_sync(gmask, pd_row, sh);
            }
            for (int c0 = 0; c0 < ld; c0 += G * VEC) {
                const int col = c0 + gl * VEC;
                const bool active = col < ld;
                double2 acc = make_double2(0.0, 0.0);
                if (!heavy) {
                    for (int64_t s = s0; s < s1; s += SPU) {
                        int jv[SPU];
                        double cv[SPU];
                        double2 xv[SPU];
#pragma unroll
                        for (int u = 0; u < SPU; ++u) {
                            const bool ok = s + u < s1;
                            jv[u] = ok ? B.idx[s + u - ib] : 0;
                            cv[u] = ok ? B.val[s + u - vb] : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < SPU; ++u) {
                            if (active && s + u < s1) {
                                const double* src = sp_src<GHOST>(a, X, jv[u], ld);
                                if (VEC == 2) xv[u] = ld2(src + col);
                                else xv[u] = make_double2(__ldg(src + col), 0.0);
                            } else {
                                xv[u] = make_double2(0.0, 0.0);
                            }
                        }
#pragma unroll
                        for (int u = 0; u < SPU; ++u) {
                            if (s + u < s1) {
                                acc.x = fma(cv[u], xv[u].x, acc.x);
                                acc.y = fma(cv[u], xv[u].y, acc.y);
                            }
                        }
                    }
                } else {
                    // dense rows: slots straight from global, G at a time, broadcast by shuffles
                    for (int64_t base = s0; base < s1; base += G) {
                        const int64_t s = base + gl;
                        int jj = 0;
                        double cc = 0.0;
                        if (s < s1) {
                            jj = __ldg(a.indices + s);
                            cc = __ldg(a.vals + s);
                        }
                        const int cnt = (int)min((int64_t)G, s1 - base);
#pragma unroll 4
                        for (int u = 0; u < cnt; ++u) {
                            const int j = __shfl_sync(gmask, jj, (lane - gl) + u);
                            const double c = __shfl_sync(gmask, cc, (lane - gl) + u);
                            if (active) {
                                if (VEC == 2) {
                                    const double* src = sp_src<GHOST>(a, X, j, ld);
                                    const double2 x = ld2(src + col);
                                    acc.x = fma(c, x.x, acc.x);
                                    acc.y = fma(c, x.y, acc.y);
                                } else {
                                    const double* src = sp_src<GHOST>(a, X, j, ld);
                                    acc.x = fma(c, __ldg(src + col), acc.x);
                                }
                            }
                        }
                    }
                }
                if (EPI >= 2) {
                    // Diagonal-constraint ADMM epilogues (per column chunk; the row dot was
                    // reduced over the whole row above).
                    const int64_t off = row * (int64_t)ld + col;
                    const double2 zr = make_double2(0.0, 0.0);
                    const double2 yv = active ? ld2cs(E.Y[0] + off) : zr;   // Wf (EPI 2) / V (EPI 3)
                    const double2 zv = active ? ld2cs(E.Z[0] + off) : zr;   // x0 (EPI 2) / U (EPI 3)
                    const double pd = pd_row;
                    const double av = __ldg(E.dmul + row);
                    double2 o = make_double2(a.alpha * acc.x, a.alpha * acc.y);
                    if (EPI == 2) {
                        // rhs = -scale C Wf + rho Wf + a (rho b - lam) Wf    (HalfStep.rhs, diagonal)
                        o = axpy2(E.ycoef[0], yv, o);
                        o = axpy2(__ldg(E.drow + row) * av, yv, o);
                        // Q = rho (a y Wf + x0), y = a <x0, Wf>   (cl_diag_cg_apply);  r = rhs - Q
                        const double cq = E.rho * (av * (av * pd));
                        const double2 q = make_double2(fma(cq, yv.x, E.rho * zv.x), fma(cq, yv.y, E.rho * zv.y));
                        double2 rr = axpy2(1.0, o, zr);
                        rr = axpy2(-1.0, q, rr);
                        if (active) {
                            st2(E.rout + off, rr);
                            if (E.cw != nullptr) st2(E.cw + off, acc);
                            dacc[0] += dot2(o, o);
                            dacc[1] += dot2(rr, rr);
                        }
                    } else {
                        // <C V, U> (objective), A(U V^T), residual, dual ascent, lam_new . b
                        if (active) dacc[0] += dot2(o, zv);
                        if (gl == 0 && c0 == 0) {
                            const double ax = 0.0 + av * pd;
                            const double bb = __ldg(E.bvec + row);
                            const double res = fma(-1.0, bb, fma(1.0, ax, 0.0));
                            const double ln = fma(E.rho, res, fma(1.0, __ldg(E.lam + row), 0.0));
                            E.axo[row] = ax;
                            E.lamo[row] = ln;
                            dacc[1] += res * res;
                            dacc[2] += ln * bb;
                        }
                    }
                    continue;
                }
                if (!active) continue;
                const int64_t off = row * (int64_t)ld + col;
                double2 o = make_double2(a.alpha * acc.x, a.alpha * acc.y);
                if (EPI == 0) {
                    if (VEC == 2) st2(a.out + off, o);
                    else a.out[off] = o.x;
                } else {
                    double2 ops[NOPS];
#pragma unroll
                    for (int j = 0; j < SP_NY; ++j) {
                        if (j < E.ny) {
                            const double2 y = VEC == 2 ? ld2cs(E.Y[j] + off) : make_double2(E.Y[j][off], 0.0);
                            ops[j] = y;
                            o = axpy2(E.ycoef[j], y, o);
                        } else {
                            ops[j] = make_double2(0.0, 0.0);
                        }
                    }
                    if (E.drow != nullptr) {
                        const double dc = __ldg(E.drow + row) * (E.dmul != nullptr ? __ldg(E.dmul + row) : 1.0);
                        o = axpy2(dc, ops[0], o);
                    }
                    if (VEC == 1) o.y = 0.0;
                    ops[SP_NY] = o;
#pragma unroll
                    for (int j = 0; j < SP_NZ; ++j) {
                        if (j < E.nz)
                            ops[SP_NY + 1 + j] = VEC == 2 ? ld2cs(E.Z[j] + off) : make_double2(E.Z[j][off], 0.0);
                        else
                            ops[SP_NY + 1 + j] = make_double2(0.0, 0.0);
                    }
                    if (a.out != nullptr) {
                        if (VEC == 2) st2(a.out + off, o);
                        else a.out[off] = o.x;
                    }
#pragma unroll
                    for (int d = 0; d < SP_ND; ++d)
                        if (d < E.ndot) dacc[d] += dot2(select2(ops, E.da[d]), select2(ops, E.db[d]));
                }
            }
        }
        __syncthreads();
    }
    if (EPI >= 1 && E.ndot > 0) reduce_and_finish<SP_ND>(dacc, E.ndot, ws, dots_out);
}

// Slot coefficients of a pattern with adjoint rows, assembled once per call
// (linops.py:100 assemble) so the SpMM reads one value per slot.
__global__ void __launch_bounds__(NT) assemble_kernel(PatDev P, int64_t nnz, double* vals) {
    for (int64_t s = (int64_t)blockIdx.x * NT + threadIdx.x; s < nnz; s += (int64_t)gridDim.x * NT)
        vals[s] = slot_coef(P, s);
}

template <int G, int VEC, int EPI, int GHOST>
int sp_blocks_per_sm() {
    static int cached = 0;
    if (cached == 0) {
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, spmm_tiled_kernel<G, VEC, EPI, GHOST>, NT, 0) !=
                cudaSuccess ||
            nb < 1)
            nb = 1;
        cached = nb;
    }
    return cached;
}

template <int G, int VEC, int EPI, int GHOST>
void sp_launch(const SpDev& a0, const EpiDev& E, double* ws, double* dots, cudaStream_t st) {
    SpDev a = a0;
    int grid = sp_blocks_per_sm<G, VEC, EPI, GHOST>() * NSM;
    if (grid > CL_RED_BLOCKS) grid = CL_RED_BLOCKS;
#if CL_SMALLN
    {   // few rows: shorter tiles so that every resident CTA gets one (latency, not staging, bounds)
        constexpr int NG = NT / G;
        const int64_t spread = (a.nrows + (int64_t)NG * grid - 1) / ((int64_t)NG * grid);
        if (spread < a.tr / NG) a.tr = (int)(spread < 1 ? 1 : spread) * NG;
    }
#endif
    a.ntiles = (a.nrows + a.tr - 1) / a.tr;
    if ((int64_t)grid > a.ntiles) grid = (int)a.ntiles;
    spmm_tiled_kernel<G, VEC, EPI, GHOST><<<grid, NT, 0, st>>>(a, E, ws, dots);
}

// 0: no ghost rows; 1: halo buffer (Xg); 2: peer memory (Xp, nown = CL_GHOST_PEERS)
static inline int sp_ghost_mode(const SpDev& a) {
    if (a.nown == CL_GHOST_PEERS) return 2;
    return a.Xg != nullptr ? 1 : 0;
}

// Ghost fields of a launch from the pattern: a halo buffer, or (nown == CL_GHOST_PEERS) a
// host table of CL_MAX_PEERS device addresses -- each rank's row block of X as mapped here,
// read now, at launch, into the kernel's parameters (so the caller may reuse the table).
static inline void sp_set_ghost(SpDev& a, const cl_pattern* S) {
    for (int k = 0; k < CL_MAX_PEERS; ++k) a.Xp[k] = nullptr;
    if (S->ghost != nullptr && S->nown == CL_GHOST_PEERS) {
        const double* const* tab = reinterpret_cast<const double* const*>(S->ghost);
        for (int k = 0; k < CL_MAX_PEERS; ++k) a.Xp[k] = tab[k];
        a.Xg = nullptr;
        a.nown = CL_GHOST_PEERS;
    } else {
        a.Xg = S->ghost;
        a.nown = S->ghost != nullptr ? (int32_t)S->nown : INT32_MAX;
    }
}

template <int G, int VEC>
void sp_dispatch_mode(int mode, const SpDev& a, const EpiDev& E, double* ws, double* dots, cudaStream_t st) {
    const int gm = sp_ghost_mode(a);
    if (mode == 2) {
        if (gm == 2) sp_launch<G, VEC, 2, 2>(a, E, ws, dots, st);
        else if (gm == 1) sp_launch<G, VEC, 2, 1>(a, E, ws, dots, st);
        else sp_launch<G, VEC, 2, 0>(a, E, ws, dots, st);
    } else {
        if (gm == 2) sp_launch<G, VEC, 3, 2>(a, E, ws, dots, st);
        else if (gm == 1) sp_launch<G, VEC, 3, 1>(a, E, ws, dots, st);
        else sp_launch<G, VEC, 3, 0>(a, E, ws, dots, st);
    }
}

template <int G, int VEC>
void sp_dispatch_epi(const SpDev& a, const EpiDev& E, double* ws, double* dots, cudaStream_t st) {
    const bool plain = E.ny == 0 && E.nz == 0 && E.ndot == 0 && E.drow == nullptr && a.out != nullptr;
    const int gm = sp_ghost_mode(a);
    if (plain) {
        if (gm == 2) sp_launch<G, VEC, 0, 2>(a, E, ws, dots, st);
        else if (gm == 1) sp_launch<G, VEC, 0, 1>(a, E, ws, dots, st);
        else sp_launch<G, VEC, 0, 0>(a, E, ws, dots, st);
    } else {
        if (gm == 2) sp_launch<G, VEC, 1, 2>(a, E, ws, dots, st);
        else if (gm == 1) sp_launch<G, VEC, 1, 1>(a, E, ws, dots, st);
        else sp_launch<G, VEC, 1, 0>(a, E, ws, dots, st);
    }
}

// ---------------------------------------------------------------------------
// single-entry constraints (constraint c = a_c (e_i e_j^T + e_j e_i^T), e.g. matrix
// completion): the half-step operator of admm.py:45 in one pass over Omega_A
// ---------------------------------------------------------------------------

// out_i = rho (sum_{slots (i,j) of c} a_c y_c Wf_j + W_i),
// y_c = a_c (W_lo . Wf_hi + W_hi . Wf_lo) with (lo, hi) = (min, max)(i, j) -- the same
// association on both rows of c, so each constraint value is computed bit-identically
// twice instead of being stored and re-read; dots[0] = <W, out>. One column chunk per
// row (ld <= 2G): lanes share the slot indices by shuffles and reduce the dots.
// ``sw``: row stride of W and Wf -- ld for separate factors, 2 ld for a pair buffer
// [W_i | Wf_i] (cl_single_entry_apply_pair), where one 16-byte-aligned 2 ld run per row holds
// both gathered operands (fewer 128-byte DRAM lines per slot, tools/micro/gather_probe.cu).
template <int G>
__global__ void SE_BOUNDS single_entry_apply_kernel(int64_t nrows, const int64_t* __restrict__ indptr,
                                                                const int32_t* __restrict__ indices,
                                                                const double* __restrict__ slot_a, int ld,
                                                                const double* __restrict__ W,
                                                                const double* __restrict__ Wf, double rho,
                                                                double* __restrict__ out, double* ws,
                                                                double* dots_out, int64_t sw) {
    double dacc[1] = {0.0};
    const int lane = threadIdx.x & 31;
    const int gl = lane % G;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane - gl));
    const int64_t groups_total = (int64_t)gridDim.x * (NT / G);
    const int col = gl * 2;
    const bool active = col < ld;
    const double2 zr = make_double2(0.0, 0.0);
    for (int64_t row = ((int64_t)blockIdx.x * NT + threadIdx.x) / G; row < nrows; row += groups_total) {
        const int64_t s0 = __ldg(indptr + row), s1 = __ldg(indptr + row + 1);
        const double2 wi = active ? ld2(W + row * sw + col) : zr;
        const double2 fi = active ? ld2(Wf + row * sw + col) : zr;
        double2 acc = zr;
        for (int64_t base = s0; base < s1; base += G) {
            const int64_t s = base + gl;
            int jj = 0;
            double aa = 0.0;
            if (s < s1) {
                jj = __ldg(indices + s);
                aa = __ldg(slot_a + s);
            }
            const int cnt = (int)min((int64_t)G, s1 - base);
            // SE_U slots at a time: their 2 SE_U row gathers are issued together, then
            // reduced one slot after another (the same arithmetic as one at a time)
            for (int u0 = 0; u0 < cnt; u0 += SE_U) {
                int jv[SE_U];
                double avv[SE_U];
                double2 wv[SE_U], fv[SE_U];
#pragma unroll
                for (int q = 0; q < SE_U; ++q) {
                    const int u = u0 + q < cnt ? u0 + q : cnt - 1;
                    jv[q] = __shfl_sync(gmask, jj, (lane - gl) + u);
                    avv[q] = __shfl_sync(gmask, aa, (lane - gl) + u);
                }
#pragma unroll
                for (int q = 0; q < SE_U; ++q) {
                    const bool ok = active && u0 + q < cnt;
                    wv[q] = ok ? ld2(W + (int64_t)jv[q] * sw + col) : zr;
                    fv[q] = ok ? ld2(Wf + (int64_t)jv[q] * sw + col) : zr;
                }
#pragma unroll
                for (int q = 0; q < SE_U; ++q) {
                    if (u0 + q >= cnt) break;
                    const int j = jv[q];
                    const double av = avv[q];
                    const double2 wj = wv[q], fj = fv[q];
                    const bool lo_is_i = row <= j;
                    double t1 = dot2(lo_is_i ? wi : wj, lo_is_i ? fj : fi);   // W_lo . Wf_hi
                    double t2 = dot2(lo_is_i ? wj : wi, lo_is_i ? fi : fj);   // W_hi . Wf_lo
#pragma unroll
                    for (int o = G / 2; o > 0; o >>= 1) {
                        t1 += __shfl_xor_sync(gmask, t1, o);
                        t2 += __shfl_xor_sync(gmask, t2, o);
                    }
                    const double y = 0.0 + av * (row == j ? t1 : t1 + t2);
                    const double coef = 0.0 + av * y;
                    acc.x = fma(coef, fj.x, acc.x);
                    acc.y = fma(coef, fj.y, acc.y);
                }
            }
        }
        if (active) {
            double2 o = make_double2(rho * acc.x, rho * acc.y);
            o = axpy2(rho, wi, o);
            st2(out + row * ld + col, o);
            dacc[0] += dot2(wi, o);
        }
    }
    reduce_and_finish<1>(dacc, 1, ws, dots_out);
}

// Halo packing for the row-sharded solve: out[i, :] = X[idx[i], :].
__global__ void __launch_bounds__(NT) gather_rows_kernel(const int32_t* __restrict__ idx, int64_t count, int h2,
                                                         const double* __restrict__ X, double* __restrict__ out) {
    const int64_t total = count * h2;
    for (int64_t k = (int64_t)blockIdx.x * NT + threadIdx.x; k < total; k += (int64_t)gridDim.x * NT) {
        const int64_t i = k / h2;
        const int q = (int)(k - i * h2);
        st2(out + 2 * k, ld2(X + 2 * ((int64_t)__ldg(idx + i) * h2 + q)));
    }
}

// ---------------------------------------------------------------------------
// CG half-step of the ADMM stage for diagonal constraints (admm.py:65/45)
// ---------------------------------------------------------------------------

struct DiagCg {
    int64_t n;
    int ld;
    const double* aval;
    double rho, beta;
    const double* r;      // p <- r + beta p first (NULL: p is read as is)
    double* p;
    const double* Wf;
    double* Q;            // NULL: only the per-row coefficients are written
    double* coef_g;       // per-row rho a_c y_c (NULL: not written)
};

// One operator application of the half-step system (admm.py:45):
//   [p <- r + beta p]   y_c = a_c <p_c, Wf_c>   Q_c = rho (a_c y_c Wf_c + p_c)   dots[0] = <p, Q>
// Rows stream through a block as one contiguous run of double2 units (as in
// diag_constraint_flat_kernel); the row dot is folded in shared memory and
// the units are finished from registers, so p and Wf are read once.
__global__ void __launch_bounds__(NT) diag_cg_apply_kernel(DiagCg a, double* ws, double* dots_out) {
    __shared__ double part[NT * DC_U];
    __shared__ double coef[NT * DC_U];
    const int h2 = a.ld >> 1;
    const int rb = flat_rows(a.n, h2);
    const int64_t nblk = (a.n + rb - 1) / rb;
    double dacc[1] = {0.0};
    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const int64_t r0 = blk * rb;
        const int nr = (int)min((int64_t)rb, a.n - r0);
        const int units = nr * h2;
        const int64_t base = r0 * (int64_t)h2;
        double2 pv[DC_U], wv[DC_U];
#pragma unroll
        for (int u = 0; u < DC_U; ++u) {
            const int e = threadIdx.x + u * NT;
            if (e < units) {
                const int64_t off = 2 * (base + e);
                wv[u] = ld2(a.Wf + off);
                if (a.r != nullptr) {
                    const double2 rv = ld2cs(a.r + off);
                    if (a.beta != 0.0) pv[u] = axpy2(a.beta, ld2cs(a.p + off), rv);
                    else pv[u] = rv;
                    st2(a.p + off, pv[u]);
                } else {
                    pv[u] = ld2cs(a.p + off);
                }
                part[e] = dot2(pv[u], wv[u]);
            }
        }
        __syncthreads();
        if (h2 <= DCF_MAXH2) {
            // short rows: one thread folds a row's unit products in order
            for (int rr = threadIdx.x; rr < nr; rr += NT) {
                double sdot = 0.0;
                for (int q = 0; q < h2; ++q) sdot += part[rr * h2 + q];
                const double av = __ldg(a.aval + r0 + rr);
                coef[rr] = a.rho * (av * (av * sdot));      // rho * a_c * y_c
                if (a.coef_g != nullptr) a.coef_g[r0 + rr] = coef[rr];
            }
        } else {
            // wide rows (high rank): a warp per row, lane-strided partial sums and a shuffle tree
            const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
            for (int rr = wid; rr < nr; rr += NWARP) {
                double sdot = 0.0;
                for (int q = lane; q < h2; q += 32) sdot += part[rr * h2 + q];
                sdot = warp_sum(sdot);
                if (lane == 0) {
                    const double av = __ldg(a.aval + r0 + rr);
                    coef[rr] = a.rho * (av * (av * sdot));
                    if (a.coef_g != nullptr) a.coef_g[r0 + rr] = coef[rr];
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < DC_U; ++u) {
            const int e = threadIdx.x + u * NT;
            if (e < units) {
                const double c = coef[e / h2];
                double2 q;
                q.x = fma(c, wv[u].x, a.rho * pv[u].x);
                q.y = fma(c, wv[u].y, a.rho * pv[u].y);
                if (a.Q != nullptr) st2(a.Q + 2 * (base + e), q);
                dacc[0] += dot2(pv[u], q);
            }
        }
        __syncthreads();
    }
    reduce_and_finish<1>(dacc, 1, ws, dots_out);
}

// CG update (admm.py:88-90): x_out = x_in + alpha p; r -= alpha Q; dots[0] = <r, r>.
__global__ void __launch_bounds__(NT) cg_step_kernel(int64_t n2, double alpha, const double* x_in, double* x_out,
                                                    const double* p, double* r, const double* Q, double* ws,
                                                    double* dots_out) {
    double dacc[1] = {0.0};
    for (int64_t k = (int64_t)blockIdx.x * NT + threadIdx.x; k < n2; k += (int64_t)gridDim.x * NT) {
        const int64_t off = 2 * k;
        st2(x_out + off, axpy2(alpha, ld2cs(p + off), ld2cs(x_in + off)));
        const double2 rv = axpy2(-alpha, ld2cs(Q + off), ld2cs(r + off));
        st2(r + off, rv);
        dacc[0] += dot2(rv, rv);
    }
    reduce_and_finish<1>(dacc, 1, ws, dots_out);
}

// cg_step with alpha = qr / *pq taken on the device (no host round trip between the
// operator application and the update). A curvature the host would reject (non-finite
// or <= 0) leaves x and r untouched; the host sees it in the same read as <r, r>.
__global__ void __launch_bounds__(NT) cg_step_dev_kernel(int64_t n2, double qr, const double* pq_ptr,
                                                        const double* x_in, double* x_out, const double* p, double* r,
                                                        const double* Q, double* ws, double* dots_out) {
    const double pq = *pq_ptr;
    if (!(isfinite(pq) && pq > 0.0)) return;
    const double alpha = qr / pq;
    double dacc[1] = {0.0};
    for (int64_t k = (int64_t)blockIdx.x * NT + threadIdx.x; k < n2; k += (int64_t)gridDim.x * NT) {
        const int64_t off = 2 * k;
        st2(x_out + off, axpy2(alpha, ld2cs(p + off), ld2cs(x_in + off)));
        const double2 rv = axpy2(-alpha, ld2cs(Q + off), ld2cs(r + off));
        st2(r + off, rv);
        dacc[0] += dot2(rv, rv);
    }
    reduce_and_finish<1>(dacc, 1, ws, dots_out);
}

// CG update with Q rebuilt from the per-row coefficients of diag_cg_apply (Q_c = coef_c Wf_c + rho p_c,
// the same expression, so bit-identical to reading a stored Q): x_out = x_in + alpha p; r -= alpha Q;
// dots[0] = <r, r>. One operand less to stream than writing Q and reading it back. alpha is taken
// from the host, or as qr / *pq on the device when pq != NULL (skip semantics of cg_step_dev).
__global__ void __launch_bounds__(NT) diag_cg_step_kernel(int64_t n, int ld, double rho, const double* coef,
                                                          const double* Wf, double alpha, double qr,
                                                          const double* pq_ptr, const double* x_in, double* x_out,
                                                          const double* p, double* r, double* ws, double* dots_out) {
    if (pq_ptr != nullptr) {
        const double pq = *pq_ptr;
        if (!(isfinite(pq) && pq > 0.0)) return;
        alpha = qr / pq;
    }
    const int h2 = ld >> 1;
    const int rb = flat_rows(n, h2);
    const int64_t nblk = (n + rb - 1) / rb;
    double dacc[1] = {0.0};
    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const int64_t r0 = blk * rb;
        const int nr = (int)min((int64_t)rb, n - r0);
        const int units = nr * h2;
        const int64_t base = r0 * (int64_t)h2;
#pragma unroll
        for (int u = 0; u < DC_U; ++u) {
            const int e = threadIdx.x + u * NT;
            if (e < units) {
                const int64_t off = 2 * (base + e);
                const double c = __ldg(coef + r0 + e / h2);
                const double2 wv = ld2cs(Wf + off);
                const double2 pv = ld2cs(p + off);
                double2 q;
                q.x = fma(c, wv.x, rho * pv.x);
                q.y = fma(c, wv.y, rho * pv.y);
                st2(x_out + off, axpy2(alpha, pv, ld2cs(x_in + off)));
                const double2 rv = axpy2(-alpha, q, ld2cs(r + off));
                st2(r + off, rv);
                dacc[0] += dot2(rv, rv);
            }
        }
    }
    reduce_and_finish<1>(dacc, 1, ws, dots_out);
}

// ADMM step end for diagonal constraints from a stored C U (written by the V half-step's
// start, cl_diag_admm_cg_init): <C U, V> (objective), A(U V^T)_c = a_c <U_c, V_c>, the
// residual, the dual ascent lam + rho (A(UV^T) - b) and lam_new . b, in one streaming pass
// instead of a second SpMM. Rows stream as in diag_cg_apply_kernel.
__global__ void __launch_bounds__(NT) diag_step_end_rows_kernel(int64_t n, int ld, const double* CU, const double* U,
                                                                const double* V, const double* aval, const double* b,
                                                                const double* lam, double rho, double* ax_out,
                                                                double* lam_out, double* ws, double* dots_out) {
    __shared__ double part[NT * DC_U];
    const int h2 = ld >> 1;
    const int rb = flat_rows(n, h2);
    const int64_t nblk = (n + rb - 1) / rb;
    double dacc[3] = {0.0, 0.0, 0.0};
    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const int64_t r0 = blk * rb;
        const int nr = (int)min((int64_t)rb, n - r0);
        const int units = nr * h2;
        const int64_t base = r0 * (int64_t)h2;
#pragma unroll
        for (int u = 0; u < DC_U; ++u) {
            const int e = threadIdx.x + u * NT;
            if (e < units) {
                const int64_t off = 2 * (base + e);
                const double2 vv = ld2cs(V + off);
                part[e] = dot2(ld2cs(U + off), vv);
                dacc[0] += dot2(ld2cs(CU + off), vv);
            }
        }
        __syncthreads();
        for (int rr = threadIdx.x; rr < nr; rr += NT) {
            double sdot = 0.0;
            for (int q = 0; q < h2; ++q) sdot += part[rr * h2 + q];
            const int64_t row = r0 + rr;
            const double ax = __ldg(aval + row) * sdot;
            const double bb = __ldg(b + row);
            const double res = ax - bb;
            const double ln = fma(rho, res, __ldg(lam + row));
            ax_out[row] = ax;
            lam_out[row] = ln;
            dacc[1] += res * res;
            dacc[2] += ln * bb;
        }
        __syncthreads();
    }
    reduce_and_finish<3>(dacc, 3, ws, dots_out);
}

// Lanczos vector updates with the scalars left on the device (spectral.py:45-61), so the
// loop needs no host round trip per step. Same arithmetic as cl_lincomb with host
// coefficients (o = fma(c_j, v_j, o) from 0 in operand order), hence bit-identical:
//   mode 0: r = u - alpha q_k [- beta q_{k-1}]     alpha = *alpha_p, beta = *beta_p
//   mode 1: q_next = (1 / sqrt(*rr_p)) r, and *beta_out = sqrt(*rr_p)
__global__ void __launch_bounds__(NT) lanczos_update_kernel(int mode, int64_t n, const double* alpha_p,
                                                            const double* beta_p, const double* u, const double* qk,
                                                            const double* qkm1, double* r, const double* rr_p,
                                                            double* beta_out, double* qn) {
    const int64_t stride = (int64_t)gridDim.x * NT;
    if (mode == 0) {
        const double na = -*alpha_p;
        const double nb = beta_p != nullptr ? -*beta_p : 0.0;
        for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += stride) {
            double o = fma(1.0, u[i], 0.0);
            o = fma(na, qk[i], o);
            if (beta_p != nullptr) o = fma(nb, qkm1[i], o);
            r[i] = o;
        }
    } else {
        const double beta = sqrt(*rr_p);
        const double cf = 1.0 / beta;
        if (blockIdx.x == 0 && threadIdx.x == 0) *beta_out = beta;
        for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += stride) qn[i] = fma(cf, r[i], 0.0);
    }
}

__global__ void __launch_bounds__(NT) gather_rows_scalar_kernel(const int32_t* __restrict__ idx, int64_t count, int ld,
                                                                const double* __restrict__ X, double* __restrict__ out) {
    const int64_t total = count * ld;
    for (int64_t k = (int64_t)blockIdx.x * NT + threadIdx.x; k < total; k += (int64_t)gridDim.x * NT) {
        const int64_t i = k / ld;
        const int q = (int)(k - i * ld);
        out[k] = __ldg(X + (int64_t)__ldg(idx + i) * ld + q);
    }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------

namespace {
int single_entry_launch(int64_t nrows, const int64_t* indptr, const int32_t* indices, const double* slot_a,
                        int32_t ld, const double* W, const double* Wf, int64_t sw, double rho, double* out,
                        double* dots_out, double* ws, void* stream) {
    if (nrows < 0 || ld < 2 || (ld & 1) || ld > 64 || indptr == nullptr || W == nullptr || Wf == nullptr ||
        out == nullptr || dots_out == nullptr || ws == nullptr)
        return CL_EARG;
    if (!aligned16(W) || !aligned16(Wf) || !aligned16(out)) return CL_EARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (nrows == 0) return (int)cudaMemsetAsync(dots_out, 0, sizeof(double), st);
    const int G = ld <= 2 ? 1 : ld <= 4 ? 2 : ld <= 8 ? 4 : ld <= 16 ? 8 : ld <= 32 ? 16 : 32;
    const int grid = red_grid(nrows * G);
#define CL_SE(GG) single_entry_apply_kernel<GG><<<grid, NT, 0, st>>>(nrows, indptr, indices, slot_a, ld, W, Wf, rho, \
                                                                   out, ws, dots_out, sw)
    switch (G) {
        case 1: CL_SE(1); break;
        case 2: CL_SE(2); break;
        case 4: CL_SE(4); break;
        case 8: CL_SE(8); break;
        case 16: CL_SE(16); break;
        default: CL_SE(32); break;
    }
#undef CL_SE
    return (int)cudaGetLastError();
}

// Pair buffer rows: P[i, half*ld : half*ld+ld] = X[i, :]   (flat row-major n x ld source)
__global__ void __launch_bounds__(NT) pair_pack_kernel(int64_t n, int h2, const double* __restrict__ X,
                                                       double* __restrict__ P, int half) {
    const int64_t total = n * h2;
    for (int64_t k = (int64_t)blockIdx.x * NT + threadIdx.x; k < total; k += (int64_t)gridDim.x * NT) {
        const int64_t i = k / h2;
        const int q = (int)(k - i * h2);
        st2(P + 2 * (i * 2 * h2 + half * h2 + q), ld2cs(X + 2 * k));
    }
}

// CG direction update of the pair path: p = r + beta p (cl_lincomb's arithmetic:
// fma(beta, p, fma(1, r, 0))), written to p and to the pair buffer's first half
__global__ void __launch_bounds__(NT) cg_direction_pair_kernel(int64_t n, int h2, double beta,
                                                               const double* __restrict__ r, double* __restrict__ p,
                                                               double* __restrict__ P) {
    const int64_t total = n * h2;
    for (int64_t k = (int64_t)blockIdx.x * NT + threadIdx.x; k < total; k += (int64_t)gridDim.x * NT) {
        const int64_t i = k / h2;
        const int q = (int)(k - i * h2);
        double2 o = axpy2(1.0, ld2cs(r + 2 * k), make_double2(0.0, 0.0));
        o = axpy2(beta, ld2cs(p + 2 * k), o);
        st2(p + 2 * k, o);
        st2(P + 2 * (i * 2 * h2 + q), o);
    }
}
}  // namespace

extern "C" {

const char* cl_version(void) { return "culorads-b200 0.1 sm_100a"; }

int cl_set_l2_fetch_granularity(int32_t bytes) {
    // L2 fetch granularity hint (0..128 bytes): random 208-byte factor-row gathers
    // over-fetch with a coarse granularity
    return (int)cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)bytes);
}

int cl_get_l2_fetch_granularity(void) {
    size_t v = 0;
    if (cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity) != cudaSuccess) return -1;
    return (int)v;
}

// Allocation base of a device address: the driver's cuMemGetAddressRange, reached
// through the runtime's entry-point table (no link-time libcuda dependency).
typedef int (*cu_range_fn)(unsigned long long* base, size_t* size, unsigned long long dptr);

static cu_range_fn cu_mem_range() {
    static cu_range_fn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<cu_range_fn>(f);
    }
    return fn;
}

int cl_ipc_export(const void* ptr, void* handle, int64_t* offset) {
    if (ptr == nullptr || handle == nullptr || offset == nullptr) return CL_EARG;
    cu_range_fn range = cu_mem_range();
    if (range == nullptr) return CL_EARG;
    unsigned long long base = 0;
    size_t size = 0;
    if (range(&base, &size, (unsigned long long)(uintptr_t)ptr) != 0) return CL_EARG;
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return (int)e;
    static_assert(sizeof(h) == CL_IPC_HANDLE_BYTES, "IPC handle size");
    memcpy(handle, &h, sizeof(h));
    *offset = (int64_t)((uintptr_t)ptr - (uintptr_t)base);
    return CL_OK;
}

int cl_ipc_import(const void* handle, void** base) {
    if (handle == nullptr || base == nullptr) return CL_EARG;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    return (int)cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess);
}

int cl_ipc_close(void* base) {
    if (base == nullptr) return CL_EARG;
    return (int)cudaIpcCloseMemHandle(base);
}

int cl_device_ok(void) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return 0;
    return p.major == 10 ? 1 : 0;
}

int cl_lincomb(const cl_lincomb_args* args, int64_t N, double* dots_out, double* ws, void* stream) {
    if (args == nullptr || N < 0 || args->nin < 0 || args->nin > CL_MAXIN) return CL_EARG;
    if (N == 0) {
        // empty operands (e.g. a rank that owns no constraints): dots are zero; torch
        // hands out NULL for 0-element tensors, so no pointer checks apply
        int nd = args->ndot;
        if (args->mode == CL_DOT_OUT_ALL && nd > 0) nd = args->nin + 1;
        if (args->mode == CL_DOT_FIRST_TWO && nd > 0) nd = 2 * CL_MAXIN - 1;
        if (nd > 0 && dots_out != nullptr)
            return (int)cudaMemsetAsync(dots_out, 0, sizeof(double) * nd, reinterpret_cast<cudaStream_t>(stream));
        return CL_OK;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    LcDev d;
    d.nin = args->nin;
    d.ndot = args->ndot;
    d.out = args->out;
    for (int j = 0; j < CL_MAXIN; ++j) {
        d.in[j] = j < args->nin ? args->in[j] : nullptr;
        d.coef[j] = j < args->nin ? args->coef[j] : 0.0;
        if (j < args->nin && (!aligned16(args->in[j]) || args->in[j] == nullptr)) return CL_EARG;
    }
    if (d.out != nullptr && !aligned16(d.out)) return CL_EARG;
    for (int j = 0; j < CL_MAXDOT; ++j) { d.da[j] = args->da[j]; d.db[j] = args->db[j]; }
    int mode = args->mode;
    if (mode < 0 || mode > 2) return CL_EARG;
    if (mode == 0 && args->ndot == 0 && args->nin > 7) mode = 1;   // plain wide combination
    if (mode == 0 && (args->nin > 7 || args->ndot > 8)) return CL_EARG;
    // input capacity of the instance (registers scale with it)
    const int nin = args->nin;
    const int kin = nin <= 2 ? 2 : nin <= 4 ? 4 : nin <= 8 ? 8 : nin <= 12 ? 12 : nin <= 17 ? 17 : CL_MAXIN;
    if (mode == 1) d.ndot = args->ndot > 0 ? args->nin + 1 : 0;
    if (mode == 2) {
        if (args->out != nullptr || args->nin < 2) return CL_EARG;
        d.ndot = args->ndot > 0 ? 2 * kin - 1 : 0;
        if (d.ndot > 0) cudaMemsetAsync(dots_out, 0, sizeof(double) * (2 * CL_MAXIN - 1),
                                        reinterpret_cast<cudaStream_t>(stream));   // the unused layout slots
    }
    if (d.ndot > 0 && (dots_out == nullptr || ws == nullptr)) return CL_EARG;
    const int64_t n2 = N / 2;
    const int tail = (int)(N & 1);
    if (N == 0) {
        if (d.ndot > 0) cudaMemsetAsync(dots_out, 0, sizeof(double) * d.ndot, st);
        return CL_OK;
    }
    switch (mode) {
#define CL_LC(M, K) lincomb_kernel<M, K><<<occ_grid((const void*)lincomb_kernel<M, K>, n2 + tail), NT, 0, st>>>( \
    d, n2, tail, ws, dots_out)
        case 0:
            if (nin <= 3) CL_LC(0, 3);
            else CL_LC(0, 7);
            break;
        case 1:
            switch (kin) {
                case 2: CL_LC(1, 2); break;
                case 4: CL_LC(1, 4); break;
                case 8: CL_LC(1, 8); break;
                case 12: CL_LC(1, 12); break;
                case 17: CL_LC(1, 17); break;
                default: CL_LC(1, CL_MAXIN); break;
            }
            break;
        default:
            switch (kin) {
                case 2:
                case 4: CL_LC(2, 4); break;
                case 8: CL_LC(2, 8); break;
                case 12: CL_LC(2, 12); break;
                case 17: CL_LC(2, 17); break;
                default: CL_LC(2, CL_MAXIN); break;
            }
#undef CL_LC
            break;
    }
    return (int)cudaGetLastError();
}

int cl_pattern_spmm(const cl_pattern* S, const double* X, int32_t ld, double alpha, const cl_epilogue* epi,
                    double* out, double* dots_out, double* ws, void* stream) {
    if (S == nullptr || X == nullptr || ld < 1 || (ld > 1 && (ld & 1))) return CL_EARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    PatDev P;
    P.nrows = S->nrows; P.indptr = S->indptr; P.indices = S->indices; P.cv = S->cv; P.c_coeff = S->c_coeff;
    P.at_ptr = S->at_ptr; P.at_con = S->at_con; P.at_val = S->at_val; P.w1 = S->w1; P.w2 = S->w2;
    P.w1g = S->w1g; P.w2g = S->w2g; P.mown = S->mown;
    EpiDev E;
    memset(&E, 0, sizeof(E));
    E.ny = 0; E.nz = 0; E.ndot = 0; E.drow = nullptr; E.dmul = nullptr;
    for (int j = 0; j < CL_MAXY; ++j) { E.Y[j] = nullptr; E.Z[j] = nullptr; E.ycoef[j] = 0.0; }
    for (int j = 0; j < 8; ++j) { E.da[j] = 0; E.db[j] = 0; }
    if (epi != nullptr) {
        if (epi->ny > CL_MAXY || epi->nz > CL_MAXY || epi->ndot > 8) return CL_EARG;
        E.ny = epi->ny; E.nz = epi->nz; E.ndot = epi->ndot;
        for (int j = 0; j < CL_MAXY; ++j) {
            E.Y[j] = epi->Y[j]; E.Z[j] = epi->Z[j]; E.ycoef[j] = epi->ycoef[j];
            if (ld > 1 && ((j < E.ny && !aligned16(E.Y[j])) || (j < E.nz && !aligned16(E.Z[j])))) return CL_EARG;
        }
        for (int j = 0; j < 8; ++j) { E.da[j] = epi->da[j]; E.db[j] = epi->db[j]; }
        E.drow = epi->drow;
        E.dmul = epi->dmul;
        if (E.drow != nullptr && E.ny < 1) return CL_EARG;
    }
    if (ld > 1 && (!aligned16(X) || (out != nullptr && !aligned16(out)))) return CL_EARG;
    if (E.ndot > 0 && (dots_out == nullptr || ws == nullptr)) return CL_EARG;
    if (P.nrows == 0) {
        if (E.ndot > 0) cudaMemsetAsync(dots_out, 0, sizeof(double) * E.ndot, st);
        return CL_OK;
    }
    int G;
    if (ld <= 2) G = 1;
    else if (ld <= 4) G = 2;
    else if (ld <= 8) G = 4;
    else if (ld <= 16) G = 8;
    else if (ld <= 32) G = 16;
    else G = 32;

    // Tiled path: one value per slot -- the objective values (c_coeff folded
    // into alpha) or the coefficients assembled into S->scratch.
    const bool need_asm = P.at_ptr != nullptr && (P.w1 != nullptr || P.w2 != nullptr);
    // (an empty pattern needs no slot values: torch hands out NULL for 0-element tensors)
    const bool tiled = ((need_asm ? S->scratch != nullptr : P.cv != nullptr) || S->nnz == 0) && S->nnz >= 0 &&
                       E.ny <= SP_NY && E.nz <= SP_NZ && E.ndot <= SP_ND &&
                       aligned16(S->indptr) && aligned16(S->indices) &&
                       (need_asm ? aligned16(S->scratch) : aligned16(P.cv));
    if (tiled) {
        // operand codes of the compact tiled epilogue: Y j -> j, out -> SP_NY, Z j -> SP_NY + 1 + j
        for (int d = 0; d < E.ndot; ++d) {
            uint8_t* c2[2] = {&E.da[d], &E.db[d]};
            for (uint8_t* c : c2) {
                if (*c == CL_OUT) *c = SP_NY;
                else if (*c >= 16) *c = (uint8_t)(SP_NY + 1 + (*c - 16));
            }
        }
        SpDev a;
        a.nrows = P.nrows; a.indptr = P.indptr; a.indices = P.indices; a.X = X; a.ld = ld; a.out = out;
        sp_set_ghost(a, S);
        if (need_asm) {
            if (S->nnz > 0) {
                int64_t g = (S->nnz + NT - 1) / NT;
                assemble_kernel<<<(int)(g > NSM * 16 ? NSM * 16 : g), NT, 0, st>>>(P, S->nnz, S->scratch);
            }
            a.vals = S->scratch;
            a.alpha = alpha;
        } else {
            a.vals = P.cv;
            a.alpha = alpha * P.c_coeff;
        }
        const int GG = (ld == 1) ? 1 : G;
        const int NG = NT / GG;
        const double avg = (double)S->nnz / (double)P.nrows;
        int rpg = (int)((0.5 * SP_SMAX) / ((avg > 1.0 ? avg : 1.0) * NG));
        const int rpg_max = (SP_PTRMAX - 4) / NG;
        if (rpg > rpg_max) rpg = rpg_max;
        if (rpg < 1) rpg = 1;
        a.tr = rpg * NG;
        a.ntiles = 0;
        if (ld == 1) {
            sp_dispatch_epi<1, 1>(a, E, ws, dots_out, st);
        } else {
            switch (G) {
                case 1: sp_dispatch_epi<1, 2>(a, E, ws, dots_out, st); break;
                case 2: sp_dispatch_epi<2, 2>(a, E, ws, dots_out, st); break;
                case 4: sp_dispatch_epi<4, 2>(a, E, ws, dots_out, st); break;
                case 8: sp_dispatch_epi<8, 2>(a, E, ws, dots_out, st); break;
                case 16: sp_dispatch_epi<16, 2>(a, E, ws, dots_out, st); break;
                default: sp_dispatch_epi<32, 2>(a, E, ws, dots_out, st); break;
            }
        }
        return (int)cudaGetLastError();
    }

    // fused-coefficient path (no scratch given, or an all-zero matrix); no ghost rows or
    // diagonal epilogue term there
    if (S->ghost != nullptr || E.drow != nullptr) return CL_EARG;
    const int64_t threads = P.nrows * G;
    const int grid = red_grid(threads);
    if (ld == 1) {
        pattern_spmm_kernel<1, 1><<<grid, NT, 0, st>>>(P, X, ld, alpha, E, out, ws, dots_out);
    } else {
        switch (G) {
            case 1: pattern_spmm_kernel<1, 2><<<grid, NT, 0, st>>>(P, X, ld, alpha, E, out, ws, dots_out); break;
            case 2: pattern_spmm_kernel<2, 2><<<grid, NT, 0, st>>>(P, X, ld, alpha, E, out, ws, dots_out); break;
            case 4: pattern_spmm_kernel<4, 2><<<grid, NT, 0, st>>>(P, X, ld, alpha, E, out, ws, dots_out); break;
            case 8: pattern_spmm_kernel<8, 2><<<grid, NT, 0, st>>>(P, X, ld, alpha, E, out, ws, dots_out); break;
            case 16: pattern_spmm_kernel<16, 2><<<grid, NT, 0, st>>>(P, X, ld, alpha, E, out, ws, dots_out); break;
            default: pattern_spmm_kernel<32, 2><<<grid, NT, 0, st>>>(P, X, ld, alpha, E, out, ws, dots_out); break;
        }
    }
    return (int)cudaGetLastError();
}

int cl_constraint_eval_halo(int64_t m, const int64_t* indptr, const int32_t* pi, const int32_t* pj,
                            const double* val, int32_t ld, const double* X1, const double* Y1, const double* X2,
                            const double* Y2, double* out1, const double* X3, const double* Y3, double* out2,
                            const double* const* ghosts, int64_t nown, void* stream);

int cl_constraint_eval(int64_t m, const int64_t* indptr, const int32_t* pi, const int32_t* pj, const double* val,
                       int32_t ld, const double* X1, const double* Y1, const double* X2, const double* Y2,
                       double* out1, const double* X3, const double* Y3, double* out2, void* stream) {
    return cl_constraint_eval_halo(m, indptr, pi, pj, val, ld, X1, Y1, X2, Y2, out1, X3, Y3, out2, nullptr, -1,
                                   stream);
}

namespace {
int constraint_eval_impl(int64_t m, const int64_t* indptr, const int32_t* pi, const int32_t* pj, const double* val,
                         int32_t ld, const double* X1, const double* Y1, const double* X2, const double* Y2,
                         double* out1, const double* X3, const double* Y3, double* out2, const double* const* ghosts,
                         int64_t nown, int64_t sx, void* stream);
}

int cl_constraint_eval_halo(int64_t m, const int64_t* indptr, const int32_t* pi, const int32_t* pj,
                            const double* val, int32_t ld, const double* X1, const double* Y1, const double* X2,
                            const double* Y2, double* out1, const double* X3, const double* Y3, double* out2,
                            const double* const* ghosts, int64_t nown, void* stream) {
    return constraint_eval_impl(m, indptr, pi, pj, val, ld, X1, Y1, X2, Y2, out1, X3, Y3, out2, ghosts, nown, 0,
                                stream);
}

int cl_constraint_eval_pair(int64_t m, const int64_t* indptr, const int32_t* pi, const int32_t* pj,
                            const double* val, int32_t ld, const double* P, double* out1, double* out2,
                            void* stream) {
    if (P == nullptr || ld < 2) return CL_EARG;
    const double* R = P;
    const double* D = P + ld;
    return constraint_eval_impl(m, indptr, pi, pj, val, ld, R, D, D, R, out1, D, D, out2, nullptr, -1,
                                2 * (int64_t)ld, stream);
}

}  // extern "C"

namespace {
int constraint_eval_impl(int64_t m, const int64_t* indptr, const int32_t* pi, const int32_t* pj, const double* val,
                         int32_t ld, const double* X1, const double* Y1, const double* X2, const double* Y2,
                         double* out1, const double* X3, const double* Y3, double* out2, const double* const* ghosts,
                         int64_t nown, int64_t sx, void* stream) {
    ConGhost gh;
    ConPeers pp;
    const bool peer = ghosts != nullptr && nown == CL_GHOST_PEERS;
    for (int k = 0; k < 6; ++k) {
        // peer mode: ghosts[k] is a HOST table of CL_MAX_PEERS row-block addresses (or NULL)
        const double* const* tab = peer ? reinterpret_cast<const double* const*>(ghosts[k]) : nullptr;
        for (int q = 0; q < CL_MAX_PEERS; ++q) pp.p[k][q] = tab != nullptr ? tab[q] : nullptr;
        gh.g[k] = ghosts != nullptr && !peer ? ghosts[k] : nullptr;
    }
    gh.nown = ghosts != nullptr ? nown : -1;
    gh.sx = sx > 0 ? sx : ld;
    if (m == 0) return CL_OK;
    if (m < 0 || ld < 1 || (ld > 1 && (ld & 1)) || X1 == nullptr || Y1 == nullptr || out1 == nullptr) return CL_EARG;
    if ((X2 == nullptr) != (Y2 == nullptr) || (X3 == nullptr) != (Y3 == nullptr)) return CL_EARG;
    if (X3 != nullptr && out2 == nullptr) return CL_EARG;
    if (m == 0) return CL_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int G = ld <= 2 ? 1 : ld <= 4 ? 2 : ld <= 8 ? 4 : ld <= 16 ? 8 : ld <= 32 ? 16 : 32;
    const int64_t threads = m * G;
    int64_t g = (threads + NT - 1) / NT;
    const int grid = (int)(g > 65535 * 8 ? 65535 * 8 : g);
    const bool one = X2 == nullptr && X3 == nullptr;
#define CL_CK(GG)                                                                                             \
    if (peer && one)                                                                                          \
        constraint_kernel<GG, 2, 1, 1><<<grid, NT, 0, st>>>(m, indptr, pi, pj, val, ld, X1, Y1, X2, Y2, out1, X3, \
                                                            Y3, out2, gh, pp);                                    \
    else if (peer)                                                                                            \
        constraint_kernel<GG, 2, 3, 1><<<grid, NT, 0, st>>>(m, indptr, pi, pj, val, ld, X1, Y1, X2, Y2, out1, X3, \
                                                            Y3, out2, gh, pp);                                    \
    else if (one)                                                                                             \
        constraint_kernel<GG, 2, 1><<<grid, NT, 0, st>>>(m, indptr, pi, pj, val, ld, X1, Y1, X2, Y2, out1, X3, Y3, \
                                                         out2, gh, pp);                                           \
    else                                                                                                      \
        constraint_kernel<GG, 2, 3><<<grid, NT, 0, st>>>(m, indptr, pi, pj, val, ld, X1, Y1, X2, Y2, out1, X3, Y3, \
                                                         out2, gh, pp)
    if (ld == 1 && peer) {
        constraint_kernel<1, 1, 3, 1><<<grid, NT, 0, st>>>(m, indptr, pi, pj, val, ld, X1, Y1, X2, Y2, out1, X3, Y3, out2,
                                                           gh, pp);
    } else if (ld == 1) {
        constraint_kernel<1, 1, 3><<<grid, NT, 0, st>>>(m, indptr, pi, pj, val, ld, X1, Y1, X2, Y2, out1, X3, Y3, out2, gh, pp);
    } else {
        switch (G) {
            case 1: CL_CK(1); break;
            case 2: CL_CK(2); break;
            case 4: CL_CK(4); break;
            case 8: CL_CK(8); break;
            case 16: CL_CK(16); break;
            default: CL_CK(32); break;
        }
    }
#undef CL_CK
    return (int)cudaGetLastError();
}
}  // namespace

extern "C" {

int cl_diag_constraint_eval(int64_t n, const double* aval, int32_t ld, const double* X1, const double* Y1,
                            const double* X2, const double* Y2, double* out1, const double* X3, const double* Y3,
                            double* out2, void* stream) {
    if (n == 0) return CL_OK;
    if (n < 0 || ld < 1 || (ld > 1 && (ld & 1)) || aval == nullptr || X1 == nullptr || Y1 == nullptr ||
        out1 == nullptr)
        return CL_EARG;
    if ((X2 == nullptr) != (Y2 == nullptr) || (X3 == nullptr) != (Y3 == nullptr)) return CL_EARG;
    if (X3 != nullptr && out2 == nullptr) return CL_EARG;
    if (n == 0) return CL_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    DiagCon d;
    d.n = n; d.aval = aval; d.ld = ld; d.nop = 0;
    d.nprod1 = X2 != nullptr ? 2 : 1;
    d.out1 = out1; d.out2 = X3 != nullptr ? out2 : nullptr;
    const double* want[6] = {X1, Y1, X2, Y2, X3, Y3};
    for (int k = 0; k < 6; ++k) {
        d.op[k] = nullptr;
        d.pidx[k] = 0;
    }
    for (int k = 0; k < 6; ++k) {
        if (want[k] == nullptr) continue;
        int f = -1;
        for (int q = 0; q < d.nop; ++q)
            if (d.op[q] == want[k]) f = q;
        if (f < 0) {
            f = d.nop++;
            d.op[f] = want[k];
        }
        d.pidx[k] = f;
    }
    // flat rows while a row's fold is short (one thread folds a row's ld/2 unit products);
    // wide rows (high rank) go to the lane-group kernel: a warp per row, a shuffle tree
    if (ld >= 2 && ld / 2 <= DCF_MAXH2 && aligned16(X1) && aligned16(Y1) && (X2 == nullptr || aligned16(X2)) &&
        (Y2 == nullptr || aligned16(Y2)) && (X3 == nullptr || aligned16(X3)) && (Y3 == nullptr || aligned16(Y3))) {
        const int rb = flat_rows(n, ld / 2);
        const int64_t nblk = (n + rb - 1) / rb;
        // one full wave of resident CTAs (the shared-memory fold limits CTAs per SM)
#define CL_DCF(NO)                                                                                  \
    diag_constraint_flat_kernel<NO><<<(int)(nblk < (int64_t)resident_blocks((const void*)diag_constraint_flat_kernel<NO>) * NSM \
                                                ? nblk                                            \
                                                : (int64_t)resident_blocks((const void*)diag_constraint_flat_kernel<NO>) * NSM), \
                                      NT, 0, st>>>(d)
        if (d.nop == 1) CL_DCF(1);
        else if (d.nop == 2) CL_DCF(2);
        else CL_DCF(6);
#undef CL_DCF
        return (int)cudaGetLastError();
    }
    const int G = ld <= 2 ? 1 : ld <= 4 ? 2 : ld <= 8 ? 4 : ld <= 16 ? 8 : ld <= 32 ? 16 : 32;
    int64_t g = (n * G + 2 * NT - 1) / (2 * NT);
    const int grid = (int)(g > NSM * 16 ? NSM * 16 : g);
#define CL_DK(GG, VV)                                                                  \
    do {                                                                               \
        if (d.nop == 1) diag_constraint_kernel<GG, VV, 1><<<grid, NT, 0, st>>>(d);     \
        else if (d.nop == 2) diag_constraint_kernel<GG, VV, 2><<<grid, NT, 0, st>>>(d); \
        else diag_constraint_kernel<GG, VV, 6><<<grid, NT, 0, st>>>(d);                \
    } while (0)
    if (ld == 1) {
        CL_DK(1, 1);
    } else {
        switch (G) {
            case 1: CL_DK(1, 2); break;
            case 2: CL_DK(2, 2); break;
            case 4: CL_DK(4, 2); break;
            case 8: CL_DK(8, 2); break;
            case 16: CL_DK(16, 2); break;
            default: CL_DK(32, 2); break;
        }
    }
#undef CL_DK
    return (int)cudaGetLastError();
}

int cl_gather_rows(const int32_t* idx, int64_t count, int32_t ld, const double* X, double* out, void* stream) {
    if (count < 0 || ld < 1 || (count > 0 && (idx == nullptr || X == nullptr || out == nullptr))) return CL_EARG;
    if (count == 0) return CL_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if ((ld & 1) || !aligned16(X) || !aligned16(out)) {
        const int64_t total = count * ld;
        int64_t g = (total + NT - 1) / NT;
        gather_rows_scalar_kernel<<<(int)(g > NSM * 16 ? NSM * 16 : g), NT, 0, st>>>(idx, count, ld, X, out);
        return (int)cudaGetLastError();
    }
    const int64_t total = count * (ld / 2);
    int64_t g = (total + NT - 1) / NT;
    gather_rows_kernel<<<(int)(g > NSM * 16 ? NSM * 16 : g), NT, 0, st>>>(idx, count, ld / 2, X, out);
    return (int)cudaGetLastError();
}

int cl_diag_cg_apply(int64_t n, int32_t ld, const double* aval, double rho, double beta, const double* r, double* p,
                     const double* Wf, double* Q, double* dots_out, double* ws, void* stream) {
    if (n < 0 || ld < 2 || (ld & 1) || ld / 2 > NT * DC_U || aval == nullptr || p == nullptr || Wf == nullptr ||
        Q == nullptr || dots_out == nullptr || ws == nullptr)
        return CL_EARG;
    if (!aligned16(p) || !aligned16(Wf) || !aligned16(Q) || (r != nullptr && !aligned16(r))) return CL_EARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (n == 0) return (int)cudaMemsetAsync(dots_out, 0, sizeof(double), st);
    DiagCg d;
    d.n = n; d.ld = ld; d.aval = aval; d.rho = rho; d.beta = beta; d.r = r; d.p = p; d.Wf = Wf; d.Q = Q;
    d.coef_g = nullptr;
    const int rb = flat_rows(n, ld / 2);
    const int64_t nblk = (n + rb - 1) / rb;
    int64_t wave = (int64_t)resident_blocks((const void*)diag_cg_apply_kernel) * NSM;
    if (wave > CL_RED_BLOCKS) wave = CL_RED_BLOCKS;
    const int grid = (int)(nblk > wave ? wave : nblk);
    diag_cg_apply_kernel<<<grid, NT, 0, st>>>(d, ws, dots_out);
    return (int)cudaGetLastError();
}

static int diag_cg_grid(const void* k, int64_t n, int32_t ld) {
    const int rb = flat_rows(n, ld / 2);
    const int64_t nblk = (n + rb - 1) / rb;
    int64_t wave = (int64_t)resident_blocks(k) * NSM;
    if (wave > CL_RED_BLOCKS) wave = CL_RED_BLOCKS;
    return (int)(nblk > wave ? wave : nblk);
}

int cl_diag_cg_apply_rows(int64_t n, int32_t ld, const double* aval, double rho, double beta, const double* r,
                          double* p, const double* Wf, double* coef, double* dots_out, double* ws, void* stream) {
    if (n < 0 || ld < 2 || (ld & 1) || ld / 2 > NT * DC_U || dots_out == nullptr || ws == nullptr) return CL_EARG;
    if (n > 0 && (aval == nullptr || p == nullptr || Wf == nullptr || coef == nullptr)) return CL_EARG;
    if (!aligned16(p) || !aligned16(Wf) || (r != nullptr && !aligned16(r))) return CL_EARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (n == 0) return (int)cudaMemsetAsync(dots_out, 0, sizeof(double), st);
    DiagCg d;
    d.n = n; d.ld = ld; d.aval = aval; d.rho = rho; d.beta = beta; d.r = r; d.p = p; d.Wf = Wf; d.Q = nullptr;
    d.coef_g = coef;
    diag_cg_apply_kernel<<<diag_cg_grid((const void*)diag_cg_apply_kernel, n, ld), NT, 0, st>>>(d, ws, dots_out);
    return (int)cudaGetLastError();
}

int cl_diag_cg_step(int64_t n, int32_t ld, double rho, const double* coef, const double* Wf, double alpha,
                    double qr, const double* pq, const double* x_in, double* x_out, const double* p, double* r,
                    double* dots_out, double* ws, void* stream) {
    if (n < 0 || ld < 2 || (ld & 1) || ld / 2 > NT * DC_U || dots_out == nullptr || ws == nullptr) return CL_EARG;
    if (n > 0 && (coef == nullptr || Wf == nullptr || x_in == nullptr || x_out == nullptr || p == nullptr ||
                  r == nullptr))
        return CL_EARG;
    if (!aligned16(Wf) || !aligned16(x_in) || !aligned16(x_out) || !aligned16(p) || !aligned16(r)) return CL_EARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (n == 0) return (int)cudaMemsetAsync(dots_out, 0, sizeof(double), st);
    diag_cg_step_kernel<<<diag_cg_grid((const void*)diag_cg_step_kernel, n, ld), NT, 0, st>>>(
        n, ld, rho, coef, Wf, alpha, qr, pq, x_in, x_out, p, r, ws, dots_out);
    return (int)cudaGetLastError();
}

int cl_cg_step(int64_t N, double alpha, const double* x_in, double* x_out, const double* p, double* r,
               const double* Q, double* dots_out, double* ws, void* stream) {
    if (N < 0 || (N & 1) || x_in == nullptr || x_out == nullptr || p == nullptr || r == nullptr || Q == nullptr ||
        dots_out == nullptr || ws == nullptr)
        return CL_EARG;
    if (!aligned16(x_in) || !aligned16(x_out) || !aligned16(p) || !aligned16(r) || !aligned16(Q)) return CL_EARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (N == 0) return (int)cudaMemsetAsync(dots_out, 0, sizeof(double), st);
    cg_step_kernel<<<occ_grid((const void*)cg_step_kernel, N / 2), NT, 0, st>>>(N / 2, alpha, x_in, x_out, p, r, Q,
                                                                                ws, dots_out);
    return (int)cudaGetLastError();
}

int cl_cg_step_dev(int64_t N, double qr, const double* pq, const double* x_in, double* x_out, const double* p,
                   double* r, const double* Q, double* dots_out, double* ws, void* stream) {
    if (N < 0 || (N & 1) || pq == nullptr || x_in == nullptr || x_out == nullptr || p == nullptr || r == nullptr ||
        Q == nullptr || dots_out == nullptr || ws == nullptr)
        return CL_EARG;
    if (!aligned16(x_in) || !aligned16(x_out) || !aligned16(p) || !aligned16(r) || !aligned16(Q)) return CL_EARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (N == 0) return (int)cudaMemsetAsync(dots_out, 0, sizeof(double), st);
    cg_step_dev_kernel<<<occ_grid((const void*)cg_step_dev_kernel, N / 2), NT, 0, st>>>(N / 2, qr, pq, x_in, x_out,
                                                                                        p, r, Q, ws, dots_out);
    return (int)cudaGetLastError();
}

// Shared setup of the fused diagonal-ADMM SpMM launches (C pattern with cv values).
static int diag_admm_launch(int mode, const cl_pattern* S, const double* X, int32_t ld, double alpha, EpiDev& E,
                            double* dots_out, double* ws, cudaStream_t st) {
    if (S == nullptr || X == nullptr || ld < 2 || (ld & 1) || dots_out == nullptr || ws == nullptr) return CL_EARG;
    if (S->at_ptr != nullptr && (S->w1 != nullptr || S->w2 != nullptr)) return CL_EARG;
    if (!(S->cv != nullptr || S->nnz == 0) || !aligned16(S->indptr) || !aligned16(S->indices) || !aligned16(X))
        return CL_EARG;
    const int G = ld <= 2 ? 1 : ld <= 4 ? 2 : ld <= 8 ? 4 : ld <= 16 ? 8 : ld <= 32 ? 16 : 32;
    SpDev a;
    a.nrows = S->nrows; a.indptr = S->indptr; a.indices = S->indices; a.vals = S->cv; a.X = X; a.ld = ld;
    a.out = nullptr; a.alpha = alpha * S->c_coeff;
    sp_set_ghost(a, S);
    const int NG = NT / G;
    const double avg = S->nrows > 0 ? (double)S->nnz / (double)S->nrows : 1.0;
    int rpg = (int)((0.5 * SP_SMAX) / ((avg > 1.0 ? avg : 1.0) * NG));
    const int rpg_max = (SP_PTRMAX - 4) / NG;
    if (rpg > rpg_max) rpg = rpg_max;
    if (rpg < 1) rpg = 1;
    a.tr = rpg * NG;
    a.ntiles = 0;
    if (S->nrows == 0) return (int)cudaMemsetAsync(dots_out, 0, sizeof(double) * E.ndot, st);
    switch (G) {
        case 1: sp_dispatch_mode<1, 2>(mode, a, E, ws, dots_out, st); break;
        case 2: sp_dispatch_mode<2, 2>(mode, a, E, ws, dots_out, st); break;
        case 4: sp_dispatch_mode<4, 2>(mode, a, E, ws, dots_out, st); break;
        case 8: sp_dispatch_mode<8, 2>(mode, a, E, ws, dots_out, st); break;
        case 16: sp_dispatch_mode<16, 2>(mode, a, E, ws, dots_out, st); break;
        default: sp_dispatch_mode<32, 2>(mode, a, E, ws, dots_out, st); break;
    }
    return (int)cudaGetLastError();
}

int cl_diag_admm_cg_init(const cl_pattern* C, const double* Wf, const double* x0, int32_t ld, double scale, double rho,
                         const double* nlam, const double* aval, double* r, double* cwf, double* dots_out, double* ws,
                         void* stream) {
    if (Wf == nullptr || x0 == nullptr || nlam == nullptr || aval == nullptr || r == nullptr) return CL_EARG;
    if (!aligned16(Wf) || !aligned16(x0) || !aligned16(r) || (cwf != nullptr && !aligned16(cwf))) return CL_EARG;
    EpiDev E;
    memset(&E, 0, sizeof(E));
    E.cw = cwf;
    E.ny = 1; E.Y[0] = Wf; E.ycoef[0] = rho;
    E.nz = 1; E.Z[0] = x0;
    E.ndot = 2;
    E.drow = nlam; E.dmul = aval; E.rho = rho; E.rout = r;
    return diag_admm_launch(2, C, Wf, ld, -scale, E, dots_out, ws, reinterpret_cast<cudaStream_t>(stream));
}

int cl_diag_admm_step_end(const cl_pattern* C, const double* U, const double* V, int32_t ld, const double* aval,
                          const double* b, const double* lam, double rho, double* ax, double* lam_new, double* dots_out,
                          double* ws, void* stream) {
    if (U == nullptr || V == nullptr || aval == nullptr || b == nullptr || lam == nullptr || ax == nullptr ||
        lam_new == nullptr)
        return CL_EARG;
    if (!aligned16(U) || !aligned16(V)) return CL_EARG;
    EpiDev E;
    memset(&E, 0, sizeof(E));
    E.ny = 1; E.Y[0] = V; E.ycoef[0] = 0.0;
    E.nz = 1; E.Z[0] = U;
    E.ndot = 3;
    E.dmul = aval; E.rho = rho; E.bvec = b; E.lam = lam; E.axo = ax; E.lamo = lam_new;
    return diag_admm_launch(3, C, V, ld, 1.0, E, dots_out, ws, reinterpret_cast<cudaStream_t>(stream));
}

int cl_diag_admm_step_end_rows(int64_t n, int32_t ld, const double* CU, const double* U, const double* V,
                               const double* aval, const double* b, const double* lam, double rho, double* ax,
                               double* lam_new, double* dots_out, double* ws, void* stream) {
    if (n < 0 || ld < 2 || (ld & 1) || ld / 2 > NT * DC_U || dots_out == nullptr || ws == nullptr) return CL_EARG;
    if (n > 0 && (CU == nullptr || U == nullptr || V == nullptr || aval == nullptr || b == nullptr ||
                  lam == nullptr || ax == nullptr || lam_new == nullptr))
        return CL_EARG;
    if (n > 0 && (!aligned16(CU) || !aligned16(U) || !aligned16(V))) return CL_EARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (n == 0) return (int)cudaMemsetAsync(dots_out, 0, 3 * sizeof(double), st);
    diag_step_end_rows_kernel<<<diag_cg_grid((const void*)diag_step_end_rows_kernel, n, ld), NT, 0, st>>>(
        n, ld, CU, U, V, aval, b, lam, rho, ax, lam_new, ws, dots_out);
    return (int)cudaGetLastError();
}


int cl_single_entry_apply(int64_t nrows, const int64_t* indptr, const int32_t* indices, const double* slot_a,
                          int32_t ld, const double* W, const double* Wf, double rho, double* out, double* dots_out,
                          double* ws, void* stream) {
    return single_entry_launch(nrows, indptr, indices, slot_a, ld, W, Wf, ld, rho, out, dots_out, ws, stream);
}

int cl_single_entry_apply_pair(int64_t nrows, const int64_t* indptr, const int32_t* indices, const double* slot_a,
                               int32_t ld, const double* P, double rho, double* out, double* dots_out, double* ws,
                               void* stream) {
    if (P == nullptr) return CL_EARG;
    return single_entry_launch(nrows, indptr, indices, slot_a, ld, P, P + ld, 2 * (int64_t)ld, rho, out, dots_out,
                               ws, stream);
}

int cl_pair_pack(int64_t n, int32_t ld, const double* X, double* P, int32_t half, void* stream) {
    if (n < 0 || ld < 2 || (ld & 1) || (half != 0 && half != 1) || X == nullptr || P == nullptr) return CL_EARG;
    if (!aligned16(X) || !aligned16(P)) return CL_EARG;
    if (n == 0) return CL_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t work = n * (ld / 2);
    pair_pack_kernel<<<occ_grid((const void*)pair_pack_kernel, work), NT, 0, st>>>(n, ld / 2, X, P, half);
    return (int)cudaGetLastError();
}

int cl_cg_direction_pair(int64_t n, int32_t ld, double beta, const double* r, double* p, double* P, void* stream) {
    if (n < 0 || ld < 2 || (ld & 1) || r == nullptr || p == nullptr || P == nullptr) return CL_EARG;
    if (!aligned16(r) || !aligned16(p) || !aligned16(P)) return CL_EARG;
    if (n == 0) return CL_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t work = n * (ld / 2);
    cg_direction_pair_kernel<<<occ_grid((const void*)cg_direction_pair_kernel, work), NT, 0, st>>>(n, ld / 2, beta, r,
                                                                                                    p, P);
    return (int)cudaGetLastError();
}

int cl_pattern_assemble(const cl_pattern* S, double* vals, void* stream) {
    if (S == nullptr || vals == nullptr || S->nnz < 0) return CL_EARG;
    if (S->nnz == 0) return CL_OK;
    PatDev P;
    memset(&P, 0, sizeof(P));
    P.nrows = S->nrows; P.indptr = S->indptr; P.indices = S->indices; P.cv = S->cv; P.c_coeff = S->c_coeff;
    P.at_ptr = S->at_ptr; P.at_con = S->at_con; P.at_val = S->at_val; P.w1 = S->w1; P.w2 = S->w2;
    P.w1g = S->w1g; P.w2g = S->w2g; P.mown = S->mown;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int64_t g = (S->nnz + NT - 1) / NT;
    assemble_kernel<<<(int)(g > NSM * 16 ? NSM * 16 : g), NT, 0, st>>>(P, S->nnz, vals);
    return (int)cudaGetLastError();
}

int cl_sddmm(int64_t K, const int32_t* imap, const int32_t* jmap, int32_t ld, const double* X, const double* Y,
             double* x, void* stream) {
    if (K < 0 || ld < 1 || (ld > 1 && (ld & 1))) return CL_EARG;
    if (K == 0) return CL_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int G = ld <= 2 ? 1 : ld <= 4 ? 2 : ld <= 8 ? 4 : ld <= 16 ? 8 : ld <= 32 ? 16 : 32;
    int64_t g = (K * G + NT - 1) / NT;
    const int grid = (int)(g > 65535 * 8 ? 65535 * 8 : g);
    if (ld == 1) { sddmm_kernel<1, 1><<<grid, NT, 0, st>>>(K, imap, jmap, ld, X, Y, x); }
    else switch (G) {
        case 1: sddmm_kernel<1, 2><<<grid, NT, 0, st>>>(K, imap, jmap, ld, X, Y, x); break;
        case 2: sddmm_kernel<2, 2><<<grid, NT, 0, st>>>(K, imap, jmap, ld, X, Y, x); break;
        case 4: sddmm_kernel<4, 2><<<grid, NT, 0, st>>>(K, imap, jmap, ld, X, Y, x); break;
        case 8: sddmm_kernel<8, 2><<<grid, NT, 0, st>>>(K, imap, jmap, ld, X, Y, x); break;
        case 16: sddmm_kernel<16, 2><<<grid, NT, 0, st>>>(K, imap, jmap, ld, X, Y, x); break;
        default: sddmm_kernel<32, 2><<<grid, NT, 0, st>>>(K, imap, jmap, ld, X, Y, x); break;
    }
    return (int)cudaGetLastError();
}

int cl_diag_alm_update(const cl_diag_update_args* a, double* dots_out, double* ws, void* stream) {
    if (a == nullptr || a->ld < 2 || (a->ld & 1) || a->nh < 0 || a->nh > CL_MAXIN) return CL_EARG;
    if (dots_out == nullptr || ws == nullptr) return CL_EARG;
    DiagDev d;
    d.n = a->n; d.ld = a->ld; d.aval = a->aval; d.tau = a->tau; d.rho = a->rho; d.scale = a->scale;
    d.R = a->R; d.D = a->D; d.CR = a->CR; d.CD = a->CD; d.ax = a->ax; d.ax_out = a->ax_out;
    d.q1 = a->q1; d.q2 = a->q2;
    d.lam = a->lam; d.b = a->b; d.g_old = a->g_old; d.g_new = a->g_new; d.y = a->y; d.nh = a->nh;
    d.refresh = a->refresh;
    for (int j = 0; j < CL_MAXIN; ++j) d.H[j] = j < a->nh ? a->H[j] : nullptr;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t n2 = a->n * (a->ld / 2);
#define CL_DU(NHH) diag_update_kernel<NHH><<<occ_grid((const void*)diag_update_kernel<NHH>, n2), NT, 0, st>>>(d, ws, dots_out)
    if (a->g_old == nullptr) {
        if (a->nh != 0) return CL_EARG;        // the first gradient has no history
        diag_update_kernel<0, false><<<occ_grid((const void*)diag_update_kernel<0, false>, n2), NT, 0, st>>>(
            d, ws, dots_out);
    } else if (a->nh == 0) CL_DU(0);
    else if (a->nh <= 4) CL_DU(4);
    else if (a->nh <= 10) CL_DU(10);
#if DU_B17
    else if (a->nh <= 17) CL_DU(17);       // 2 * memory + 1 at the default L-BFGS memory 8
#endif
    else CL_DU(CL_MAXIN);
#undef CL_DU
    return (int)cudaGetLastError();
}

int cl_lanczos_update(int32_t mode, int64_t n, const double* alpha, const double* beta, const double* u,
                      const double* qk, const double* qkm1, double* r, const double* rr, double* beta_out, double* qn,
                      void* stream) {
    if (n < 0 || (mode != 0 && mode != 1)) return CL_EARG;
    if (mode == 0 && (alpha == nullptr || u == nullptr || qk == nullptr || r == nullptr ||
                      (beta != nullptr && qkm1 == nullptr)))
        return CL_EARG;
    if (mode == 1 && (rr == nullptr || beta_out == nullptr || r == nullptr || qn == nullptr)) return CL_EARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t nb = (n + NT - 1) / NT;
    const int grid = (int)(nb < 1 ? 1 : (nb > NSM * 8 ? NSM * 8 : nb));
    lanczos_update_kernel<<<grid, NT, 0, st>>>(mode, n, alpha, beta, u, qk, qkm1, r, rr, beta_out, qn);
    return (int)cudaGetLastError();
}

int cl_basis_project(const double* Q, int64_t ldq, int32_t k_cnt, int64_t n, const double* v, double* h, double* ws,
                     void* stream) {
    if (k_cnt < 0 || (int64_t)k_cnt * BP_CHUNKS > CL_WS_DOUBLES) return CL_EARG;
    if (k_cnt == 0) return CL_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    dim3 grid(BP_CHUNKS, (k_cnt + BP_TILE - 1) / BP_TILE);
    basis_project_kernel<<<grid, NT, 0, st>>>(Q, ldq, k_cnt, n, v, ws);
    basis_project_finish<<<(k_cnt + 3) / 4, 128, 0, st>>>(ws, BP_CHUNKS, k_cnt, h);
    return (int)cudaGetLastError();
}

int cl_basis_subtract(const double* Q, int64_t ldq, int32_t k_cnt, int64_t n, const double* h, double* v,
                      void* stream) {
    if (k_cnt < 0 || k_cnt > 4096) return CL_EARG;
    if (k_cnt == 0 || n == 0) return CL_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int64_t g = (n + NT - 1) / NT;
    const int grid = (int)(g > NSM * 16 ? NSM * 16 : g);
    basis_subtract_kernel<<<grid, NT, k_cnt * sizeof(double), st>>>(Q, ldq, k_cnt, n, h, v);
    return (int)cudaGetLastError();
}

}  // extern "C"
