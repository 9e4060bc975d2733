// smoe_kernels.cuh -- sm_100a device code of the Rasterized SMoE hot path.
//
// Citations: P:n = PAPER.md line n (arxiv 2510.05814), S:n = SPEC.md line n,
// Q-numbers = readings in DESIGN.md.  Pipeline of one step:
//
//   k_preprocess  per kernel: whitening record, square 99% box,
//                 per-block overlap counts (atomics); the last CTA
//                 scans the counts into block ranges               [§8(a) a1, a2]
//   k_scatter     kernel ids into their blocks' buckets           [a3]
//   k_raster      per 16x16 block: bucket sort by kernel id (second
//                 radix digit), forward, loss, backward            [a4-a7, a9]
//   k_adam        chain rule -> Adam -> clamp, accumulator reset   [a8]
//
// The binning is an MSD radix sort of the key (tile_id | kernel_id): the
// first digit (the whole tile id) is a counting sort driven by per-block
// atomics, the second (kernel id) an in-shared-memory sort per bucket.  The
// result is the canonical list K_n (Eq. 5): blocks ascending, kernel ids
// ascending inside a block (Q18).
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <limits.h>
#include <type_traits>
#include <cstdio>

namespace smoe {

constexpr int TILE = 16;                 // 16x16 blocks
// build-time tuning knobs (A/B builds in scripts/; defaults are the tuned values)
#ifndef SMOE_FWD_UNROLL
#define SMOE_FWD_UNROLL 1                // forward kernel-loop unroll (x4 constant experts, x2 kernel-parallel train)
#endif
#ifndef SMOE_KPAR_MINB
#define SMOE_KPAR_MINB 6                 // kernel-parallel raster, linear experts: min CTAs/SM
#endif
#ifndef SMOE_KPAR_MINB_CONST
#define SMOE_KPAR_MINB_CONST 7           // ... constant experts (fewer live sums, no spills at 7)
#endif
#ifndef SMOE_RASTER_BATCH
#define SMOE_RASTER_BATCH 128            // kernel records staged per shared-memory batch
#endif
#ifndef SMOE_PRE_ATOM
#define SMOE_PRE_ATOM 4                  // direct binning: count atomics in flight per kernel
#endif
#ifndef SMOE_FWD_PREFETCH
#define SMOE_FWD_PREFETCH 0              // forward: load record j+1's test half while testing record j
                                         // (measured: +2 registers cost a resident CTA, -9% config 3)
#endif
// Device bounds checks of the debug build (-DSMOE_DEBUG; `make variant
// NAME=dbg EXTRA=-DSMOE_DEBUG`): a failed check prints its site and traps,
// so the calling test fails with a CUDA error.  Used in place of
// compute-sanitizer where the tool is unavailable.
#ifdef SMOE_DEBUG
#define SMOE_CHECK(c)                                                                    \
    do {                                                                                 \
        if (!(c)) {                                                                      \
            printf("SMOE_CHECK failed at %s:%d: %s\n", __FILE__, __LINE__, #c);          \
            __trap();                                                                    \
        }                                                                                \
    } while (0)
#else
#define SMOE_CHECK(c) \
    do {              \
    } while (0)
#endif
#ifndef SMOE_SEED_SOA
#define SMOE_SEED_SOA 1                  // backward seeds as 32-bit SoA: conflict-free loads of random pixel slots
                                         // (config 3 raster 264.5 -> 259.1 us, config 2 48.6 -> 47.0 us; the
                                         // 16-byte slot layout carried 85% of the raster's bank-conflict wavefronts)
#endif
#ifndef SMOE_R4_XF
#define SMOE_R4_XF 1                     // four-pixel render: cull test on block-centred records (constant experts)
#endif
#ifndef SMOE_BWD_PACK
#define SMOE_BWD_PACK 0                  // kernel-parallel backward: raw sums kept as f32x2 pixel-pair
                                         // accumulators (bit 0: expert sums, bit 1: geometric sums);
                                         // 0 (scalar) measured fastest: the pairs cost a resident CTA
#endif
constexpr int kFwdUnroll = SMOE_FWD_UNROLL;

// 128-bit shared load from a 32-bit shared-window address (keeps the
// generic-to-shared conversion out of the backward loop)
__device__ __forceinline__ float4 lds128(unsigned a)
{
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ float2 lds64(unsigned a)
{
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ int lds32(unsigned a)
{
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
constexpr int PRE_ATOM = SMOE_PRE_ATOM;
constexpr float LOG2E = 1.4426950408889634f;
constexpr unsigned FULL = 0xffffffffu;
constexpr int SORT_CAP = 2048;           // bucket size sorted in one smem pass

// Per-grid device counters (one block grid = one raster: the training image
// or one render resolution).
struct GridCtr {
    long long pairs;      // P of the most recent binning on this grid
    long long need;       // latched: largest P (CSR) / longest bucket (direct) beyond the capacity
    long long skipped;    // latched: sequences skipped because of overflow
    unsigned int ticket;  // last-CTA ticket of k_preprocess
    unsigned int work;    // raster work-queue head (reset by k_preprocess)
    unsigned int scan_vid;   // k_scan_lookback: virtual CTA counter
    unsigned int scan_done;  // k_scan_lookback: finished-CTA ticket
    unsigned int epoch;      // k_scan_lookback: tag of the current scan
    unsigned int skip;       // 1: the last binning overflowed its capacity (consumers skip)
    unsigned long long acc_pairs;  // direct buckets: pairs emitted by this binning (CTA sums)
    int acc_max;             // direct buckets: longest bucket of this binning
    int pad2;
};

// Per-handle device counters.
struct HandleCtr {
    long long t;          // Adam step counter (1-based after the first step)
    long long nonfinite;  // latched non-finite flag (S:355 DivergedLoss)
    unsigned int done;    // last-block ticket of k_adam
    unsigned int pad;
};

struct ParamsDev {
    const float *mu, *chol, *log_pi, *expert;
};
struct ParamsMut {
    float *mu, *chol, *log_pi, *expert;
};
struct LrDev {
    float mu, chol, log_pi, expert, slope;
};

// Record stride (floats) of the per-kernel render record:
// [mu_x, mu_y, a, b, c, log_pi*log2e, expert(C*E)] padded to float4.
template <int C, int E>
struct Rec {
    static constexpr int P = 6 + C * E;          // parameters per kernel
    static constexpr int RS = (P + 3) & ~3;      // record stride, floats
    static constexpr int V = P <= 8 ? 8 : 16;    // accumulator stride (pow2)
};

__device__ __forceinline__ float ex2_approx(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ bool finitef(float x) { return isfinite(x); }

// gpu-scope acq_rel add (one release of the CTA's prior writes after a
// barrier, one acquire for what follows; cheaper than __threadfence(), a
// sequentially consistent fence plus an L1 invalidation)
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned *p, unsigned v)
{
    unsigned r;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
    return r;
}

// ------------------------------------------------------------ a2 / a4 -----
// Exclusive scan of the per-block counts by one CTA of NT threads (4 counts
// per thread per round).  Produces start[n+1] and the scatter cursors, zeroes
// the counts for the next binning, publishes P and latches overflow; also
// zeroes the loss partials consumed by the raster that follows.  Run by the
// last CTA of k_preprocess to finish (all count atomics are visible then).
template <int NT>
__device__ __forceinline__ void scan_counts(int *__restrict__ cnt, int n, int *__restrict__ start,
                                            int *__restrict__ cursor, long long cap, GridCtr *gc,
                                            double *dstats)
{
    constexpr int NW = NT / 32;
    __shared__ int warp_tot[NW];
    __shared__ long long carry_s;
    int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) carry_s = 0;
    if (tid < 4 && dstats) dstats[tid] = 0.0;
    __syncthreads();
    for (int base = 0; base < n; base += 4 * NT) {
        int i0 = base + tid * 4;
        int v[4];
#pragma unroll
        for (int q = 0; q < 4; q++) v[q] = (i0 + q < n) ? __ldcg(cnt + i0 + q) : 0;
        int loc = v[0] + v[1] + v[2] + v[3];
        int incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) warp_tot[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            int w = lane < NW ? warp_tot[lane] : 0;
            int wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int t = __shfl_up_sync(FULL, wi, o);
                if (lane >= o) wi += t;
            }
            if (lane < NW) warp_tot[lane] = wi - w;  // exclusive
        }
        __syncthreads();
        long long carry = carry_s;
        int ex = (int)carry + warp_tot[wid] + incl - loc;
#pragma unroll
        for (int q = 0; q < 4; q++) {
            if (i0 + q < n) {
                start[i0 + q] = ex;
                cursor[i0 + q] = ex;
                cnt[i0 + q] = 0;
            }
            ex += v[q];
        }
        __syncthreads();
        if (tid == NT - 1) carry_s = carry + warp_tot[NW - 1] + incl;
        __syncthreads();
    }
    if (tid == 0) {
        long long P = carry_s;
        start[n] = (int)P;
        gc->pairs = P;
        gc->skip = P > cap ? 1u : 0u;
        if (P > cap) {
            if (P > gc->need) gc->need = P;
            gc->skipped += 1;
        }
    }
}

// ------------------------------------------------------- box modes -------
// Reading Q4: 0 square box of half side R sqrt(lambda_max)
// (default), 1 the ellipse's axis-aligned box (half sides
// R sqrt(Sigma_xx), R sqrt(Sigma_yy)), 2 exact: the mode-1 blocks whose
// rectangle of pixel-centre sample points meets the ellipse.  Every mode
// lists each block holding a pixel inside the ellipse (pixels do not depend
// on it); the lists shrink from mode 0 to 2 for anisotropic kernels.
struct BoxGeo {
    int mode;          // 0 square, 1 aabb, 2 exact
    float isx, isy;    // source spacing of output samples: x = (j + 1/2) isx - 1/2
    int oW, oH;
};

// min over the block's pixel-centre rectangle of d^2 = u^2 + v^2
// (u = a dx, v = b dx + c dy), compared with R2 -- mode 2's block test
__device__ __forceinline__ bool block_meets(float mux, float muy, float a, float b, float c, int tx, int ty,
                                            const BoxGeo &G, float R2)
{
    const float x0 = (TILE * tx + 0.5f) * G.isx - 0.5f, x1 = (min(TILE * tx + TILE - 1, G.oW - 1) + 0.5f) * G.isx - 0.5f;
    const float y0 = (TILE * ty + 0.5f) * G.isy - 0.5f, y1 = (min(TILE * ty + TILE - 1, G.oH - 1) + 0.5f) * G.isy - 0.5f;
    if (mux >= x0 && mux <= x1 && muy >= y0 && muy <= y1) return true;
    // Q(dx, dy) = p dx^2 + 2 q dx dy + r dy^2
    const float pp = a * a + b * b, qq = b * c, rr = c * c;
    float best = INFINITY;
#pragma unroll
    for (int e = 0; e < 2; e++) {
        float dx = (e ? x1 : x0) - mux;
        float dy = fminf(fmaxf(-qq * dx / rr, y0 - muy), y1 - muy);
        best = fminf(best, pp * dx * dx + 2.f * qq * dx * dy + rr * dy * dy);
        dy = (e ? y1 : y0) - muy;
        dx = fminf(fmaxf(-qq * dy / pp, x0 - mux), x1 - mux);
        best = fminf(best, pp * dx * dx + 2.f * qq * dx * dy + rr * dy * dy);
    }
    return best <= R2;
}

// ---------------------------------------------------------------- a1 ------
// Geometry shader: Sigma = L L^T, lambda_max in closed form,
// square box of half side r = sqrt(R2 lambda_max), pixel-centre rule (Q5)
// on the out_H x out_W raster, then the per-block overlap counts for the
// block rows [ty_lo, ty_hi) (the whole grid, or one multi-GPU band).
// Whitening: u = a dx, v = b dx + c dy with a = 1/l11, b = -l21/(l11 l22),
// c = 1/l22, so d^2 = u^2 + v^2 = delta^T Sigma^-1 delta.
// Record (whitening, log2 pi, experts) and tile box of one kernel from its
// parameter values; shared by the binning kernels and the fused Adam epilogue
// (which writes the next step's records from the parameters it just
// updated).  Returns the inclusive block box {x0, x1, y0, y1} of the raster,
// or -1s when the kernel covers no pixel centre or a value is not finite.
template <int C, int E>
__device__ __forceinline__ int4 record_box(float2 mu, float l11, float l21, float l22, float lp, const float *ex,
                                           float R2, float sx, float sy, int oW, int oH, int mode,
                                           float (&r)[Rec<C, E>::RS], bool &ok)
{
    using R = Rec<C, E>;
    float a = 1.0f / l11, c = 1.0f / l22;
    float b = -l21 / (l11 * l22);
    r[0] = mu.x; r[1] = mu.y; r[2] = a; r[3] = b; r[4] = c; r[5] = lp * LOG2E;
    ok = finitef(mu.x) && finitef(mu.y) && finitef(a) && finitef(b) && finitef(c) && finitef(lp);
#pragma unroll
    for (int i = 0; i < C * E; i++) {
        r[6 + i] = ex[i];
        ok = ok && finitef(r[6 + i]);
    }
#pragma unroll
    for (int i = R::P; i < R::RS; i++) r[i] = 0.0f;
    float s11 = l11 * l11, s12 = l11 * l21, s22 = l21 * l21 + l22 * l22;
    float rx, ry;
    if (mode == 0) {
        float h = 0.5f * (s11 - s22);
        float lmax = 0.5f * (s11 + s22) + sqrtf(h * h + s12 * s12);
        rx = ry = sqrtf(R2 * lmax);
    } else {
        rx = sqrtf(R2 * s11);
        ry = sqrtf(R2 * s22);
    }
    float xl = ceilf((mu.x - rx + 0.5f) * sx - 0.5f);
    float xh = floorf((mu.x + rx + 0.5f) * sx - 0.5f);
    float yl = ceilf((mu.y - ry + 0.5f) * sy - 0.5f);
    float yh = floorf((mu.y + ry + 0.5f) * sy - 0.5f);
    xl = fmaxf(xl, 0.0f); yl = fmaxf(yl, 0.0f);
    xh = fminf(xh, (float)(oW - 1)); yh = fminf(yh, (float)(oH - 1));
    if (ok && xl <= xh && yl <= yh) return make_int4((int)xl / TILE, (int)xh / TILE, (int)yl / TILE, (int)yh / TILE);
    return make_int4(-1, -1, -1, -1);
}

// Destination of the fused Adam epilogue's records (training grid, current
// band, lscale 1); rec == nullptr: no records (standalone binning follows).
struct RecOut {
    float *rec;
    int4 *tbox;
    float R2;
    int oW, oH, ty_lo, ty_hi, mode;
    int K;   // pool size (debug bounds checks)
};

template <int C, int E>
__device__ __forceinline__ void write_record(const RecOut &ro, int k, float2 mu, float l11, float l21, float l22,
                                             float lp, const float *ex, HandleCtr *hc)
{
    using R = Rec<C, E>;
    float r[R::RS];
    bool ok;
    const int4 tb = record_box<C, E>(mu, l11, l21, l22, lp, ex, ro.R2, 1.0f, 1.0f, ro.oW, ro.oH, ro.mode, r, ok);
    if (!ok) atomicExch((unsigned long long *)&hc->nonfinite, 1ull);
    if (tb.x >= 0 && max(tb.z, ro.ty_lo) <= min(tb.w, ro.ty_hi - 1)) {
        float4 *dst = reinterpret_cast<float4 *>(ro.rec) + (size_t)k * (R::RS / 4);
#pragma unroll
        for (int q = 0; q < R::RS / 4; q++) dst[q] = make_float4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
    }
    SMOE_CHECK(k >= 0 && k < ro.K);
    ro.tbox[k] = tb;
}

template <int C, int E>
__device__ __forceinline__ void
preprocess_one(int k, ParamsDev p, float R2, float sx, float sy, int oW, int oH,
               int nx, int ty_lo, int ty_hi, float *__restrict__ rec,
               int4 *__restrict__ tbox, int *__restrict__ cnt, HandleCtr *hc, float lscale, int mode,
               bool direct = false, int *__restrict__ dids = nullptr, int bcap = 0,
               int *n_emit = nullptr, int *max_len = nullptr, int sub = 0, int tpk = 1)
{
    // tpk threads per kernel (direct buckets, small pools): thread `sub`
    // emits the kernel's blocks sub, sub + tpk, ...; thread 0 alone writes
    // the record, the tile box and the non-finite flag
    using R = Rec<C, E>;
    float2 mu = reinterpret_cast<const float2 *>(p.mu)[k];
    // lscale = sqrt(s) applies the sharpening edit Sigma -> s Sigma (render only)
    float l11 = p.chol[3 * k] * lscale, l21 = p.chol[3 * k + 1] * lscale, l22 = p.chol[3 * k + 2] * lscale;
    float lp = p.log_pi[k];
    float r[R::RS];
    bool ok;
    const int4 tb = record_box<C, E>(mu, l11, l21, l22, lp, p.expert + (size_t)k * C * E, R2, sx, sy, oW, oH, mode, r, ok);
    if (!ok && sub == 0) atomicExch((unsigned long long *)&hc->nonfinite, 1ull);
    const float a = r[2], b = r[3], c = r[4];
    const BoxGeo G{mode, 1.0f / sx, 1.0f / sy, oW, oH};
    if (tb.x >= 0) {
        int y0 = max(tb.z, ty_lo), y1 = min(tb.w, ty_hi - 1);
        // the record is read only through the block lists: write it only for
        // a kernel listed in some block of the band (a multi-GPU rank skips
        // the records of kernels outside its band)
        if (y0 <= y1 && sub == 0) {
            float4 *dst = reinterpret_cast<float4 *>(rec) + (size_t)k * (R::RS / 4);
#pragma unroll
            for (int q = 0; q < R::RS / 4; q++) dst[q] = make_float4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
        }
        if (direct) {
            // direct buckets: the count atomic returns k's slot in block t's
            // fixed-capacity bucket (PRE_ATOM atomics in flight per round)
            const int wx = tb.y - tb.x + 1, nbx = max(0, y1 - y0 + 1) * wx;
            int emitted = 0;
            for (int i0 = sub; i0 < nbx; i0 += PRE_ATOM * tpk) {
                int t[PRE_ATOM], sl[PRE_ATOM];
                bool on[PRE_ATOM];
#pragma unroll
                for (int q = 0; q < PRE_ATOM; q++) {
                    const int i = i0 + q * tpk, yy = y0 + i / wx, xx = tb.x + i % wx;
                    t[q] = yy * nx + xx;
                    on[q] = i < nbx && (mode != 2 || block_meets(mu.x, mu.y, a, b, c, xx, yy, G, R2));
                    sl[q] = on[q] ? atomicAdd(&cnt[t[q]], 1) : bcap;
                }
#pragma unroll
                for (int q = 0; q < PRE_ATOM; q++) {
                    SMOE_CHECK(!on[q] || (t[q] >= ty_lo * nx && t[q] < ty_hi * nx));
                    if (sl[q] < bcap) dids[(size_t)t[q] * bcap + sl[q]] = k;
                    if (on[q]) { *max_len = max(*max_len, sl[q] + 1); emitted++; }
                }
            }
            *n_emit = emitted;
        } else if (cnt) {
            for (int ty = y0; ty <= y1; ty++)
                for (int tx = tb.x; tx <= tb.y; tx++)
                    if (mode != 2 || block_meets(mu.x, mu.y, a, b, c, tx, ty, G, R2)) atomicAdd(&cnt[ty * nx + tx], 1);
        }
    }
    if (sub == 0) tbox[k] = tb;
}

constexpr int PRE_NT = 256;

// Direct buckets (a1 + a3 in one pass): kernel k's id went straight into the
// slot its count atomic returned in block t's fixed-capacity bucket
// ids[t * bcap, ...).  The count array is the bucket-length array: the
// raster CTA of block t reads it and resets it (no pass over the blocks
// here).  Every CTA adds its pair count and longest slot to the grid
// counters; the last CTA of k_preprocess publishes P, latches overflow (a
// bucket longer than bcap: consumers skip, the host regrows), and zeroes the
// loss partials.
__device__ __forceinline__ void finish_direct(int bcap, GridCtr *gc, double *dstats)
{
    if (threadIdx.x < 4 && dstats) dstats[threadIdx.x] = 0.0;
    if (threadIdx.x == 0) {
        const long long P = (long long)__ldcg(&gc->acc_pairs);
        const int mx = __ldcg(&gc->acc_max);
        gc->acc_pairs = 0ull;
        gc->acc_max = 0;
        gc->pairs = P;
        const bool ovf = mx > bcap;
        gc->skip = ovf ? 1u : 0u;
        if (ovf) {
            if (mx > gc->need) gc->need = mx;
            gc->skipped += 1;
        }
    }
}

#ifndef SMOE_PRE_MINB
#define SMOE_PRE_MINB 1      // k_preprocess: min resident CTAs per SM (register cap; 6 and 8 spill and lose 12-16%)
#endif
template <int C, int E>
__global__ void __launch_bounds__(PRE_NT, SMOE_PRE_MINB)
k_preprocess(int K, ParamsDev p, float R2, float sx /* oW/W */, float sy /* oH/H */, int oW, int oH,
             int nx, int ty_lo, int ty_hi, float *__restrict__ rec,
             int4 *__restrict__ tbox, int *__restrict__ cnt, HandleCtr *hc,
             int n_tiles, int *__restrict__ start, int *__restrict__ cursor, long long cap,
             GridCtr *gc, double *dstats, int *__restrict__ order, float lscale, int build_order,
             int *__restrict__ dids, int bcap, int *__restrict__ len, int mode, int tpk)
{
    // tpk > 1 (direct buckets, small pools): tpk consecutive threads share a
    // kernel and split its block atomics -- more CTAs in flight and fewer
    // dependent atomic rounds per thread (the small-pool latency floor)
    const int gt = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = gt / tpk, sub = gt - k * tpk;
    int n_emit = 0, max_len = 0;
    if (k < K)
        preprocess_one<C, E>(k, p, R2, sx, sy, oW, oH, nx, ty_lo, ty_hi, rec, tbox, cnt, hc, lscale, mode,
                             len != nullptr, dids, bcap, &n_emit, &max_len, sub, tpk);
    if (len) {
        // direct buckets: this CTA's pairs and longest slot to the grid counters
        __shared__ unsigned long long s_pairs;
        __shared__ int s_max;
        if (threadIdx.x == 0) { s_pairs = 0ull; s_max = 0; }
        __syncthreads();
        unsigned long long pe = (unsigned)n_emit;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            pe += __shfl_xor_sync(FULL, pe, o);
            max_len = max(max_len, __shfl_xor_sync(FULL, max_len, o));
        }
        if ((threadIdx.x & 31) == 0) {
            if (pe) atomicAdd(&s_pairs, pe);
            if (max_len) atomicMax(&s_max, max_len);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (s_pairs) atomicAdd(&gc->acc_pairs, s_pairs);
            if (s_max) atomicMax(&gc->acc_max, s_max);
        }
    }
    if (!order && !len) return;   // large grid: k_scan_lookback follows
    // the last CTA to finish publishes the grid's totals (a2)
    // (grid-sync pattern: barrier, then one acq_rel ticket by thread 0; the
    // last CTA reads the counters from L2)
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) last = atom_add_acq_rel_gpu(&gc->ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    if (len) {
        finish_direct(bcap, gc, dstats);
        if (threadIdx.x == 0) { gc->ticket = 0; gc->work = 0; }
        return;
    }
    scan_counts<PRE_NT>(cnt, n_tiles, start, cursor, cap, gc, dstats);
    if (!build_order) {
        if (threadIdx.x == 0) { gc->ticket = 0; gc->work = 0; }
        return;
    }
    // raster work order for the band's blocks: longest lists first (LPT),
    // counting sort on min(|K_n|, 255)
    __shared__ int hist[256];
    const int t0 = ty_lo * nx, nt = (ty_hi - ty_lo) * nx;
    hist[threadIdx.x] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < nt; i += PRE_NT) {
        int c = start[t0 + i + 1] - start[t0 + i];
        atomicAdd(&hist[255 - min(c, 255)], 1);
    }
    __syncthreads();
    {
        int v = hist[threadIdx.x], inc = v, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += t;
        }
        __shared__ int wt[PRE_NT / 32];
        if (lane == 31) wt[wid] = inc;
        __syncthreads();
        int pre = 0;
        for (int w = 0; w < wid; w++) pre += wt[w];
        hist[threadIdx.x] = pre + inc - v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nt; i += PRE_NT) {
        int c = start[t0 + i + 1] - start[t0 + i];
        int pos = atomicAdd(&hist[255 - min(c, 255)], 1);
        order[pos] = t0 + i;
    }
    if (threadIdx.x == 0) { gc->ticket = 0; gc->work = 0; }
}


// ------------------------------------------- a1 + a3, large pools -------
// Two-stage direct-bucket binning for large pools (K >= PERM_MIN_K).  The
// one-pass form (k_preprocess) issues one returning global atomic per
// (kernel, block) pair: 8.35 M at config 5, the throughput limit of that
// kernel (ncu: long-scoreboard stalls on the returning atomics).  Here
//   stage 1  k_records: per kernel in id order (coalesced), the record and
//            the tile box -- no atomics;
//   stage 2  k_emit: per kernel in a spatially sorted order (perm), the CTA
//            counts its kernels' (block) entries in a shared-memory window
//            of blocks, adds each window block's count to the block's global
//            counter with ONE returning atomic, and hands out slots from the
//            returned base with shared-memory atomics.
// The permutation only groups kernels that are close in the image (a
// counting sort of the centres into ~256-kernel spatial buckets, refreshed
// every PERM_REFRESH binnings; centres move by <= lr_mu ~ 0.01 px per step);
// any permutation gives the same lists, because the raster sorts each bucket
// by kernel id (a4).
constexpr int PERM_NT = 1024;           // single-CTA scan of the bucket histogram
constexpr int PERM_MAX_BUCKETS = 16384;
constexpr int EMIT_NT = 256;
constexpr int EMIT_WIN = 2048;          // shared window of blocks per CTA

__device__ __forceinline__ int perm_key(float2 mu, float bx_scale, float by_scale, int nbx, int nby)
{
    // spatial bucket of the centre (clamped; non-finite centres to bucket 0)
    float fx = mu.x * bx_scale, fy = mu.y * by_scale;
    int bx = (fx == fx) ? (int)fminf(fmaxf(fx, 0.f), (float)(nbx - 1)) : 0;
    int by = (fy == fy) ? (int)fminf(fmaxf(fy, 0.f), (float)(nby - 1)) : 0;
    return by * nbx + bx;
}

__global__ void __launch_bounds__(256)
k_perm_count(int K, const float *__restrict__ mu, float bx_scale, float by_scale, int nbx, int nby,
             int *__restrict__ hist)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < K) atomicAdd(&hist[perm_key(reinterpret_cast<const float2 *>(mu)[k], bx_scale, by_scale, nbx, nby)], 1);
}

// exclusive scan of nb <= PERM_MAX_BUCKETS counts by one CTA, in place
__global__ void __launch_bounds__(PERM_NT)
k_perm_scan(int *__restrict__ hist, int nb)
{
    constexpr int PER = PERM_MAX_BUCKETS / PERM_NT;
    __shared__ int wsum[PERM_NT / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int v[PER], loc = 0;
#pragma unroll
    for (int q = 0; q < PER; q++) {
        const int i = tid * PER + q;
        v[q] = i < nb ? hist[i] : 0;
        loc += v[q];
    }
    int inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        const int w = wsum[lane];
        int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(FULL, wi, o);
            if (lane >= o) wi += t;
        }
        wsum[lane] = wi - w;
    }
    __syncthreads();
    int e = wsum[wid] + inc - loc;
#pragma unroll
    for (int q = 0; q < PER; q++) {
        const int i = tid * PER + q;
        if (i < nb) hist[i] = e;
        e += v[q];
    }
}

__global__ void __launch_bounds__(256)
k_perm_scatter(int K, const float *__restrict__ mu, float bx_scale, float by_scale, int nbx, int nby,
               int *__restrict__ cursor, int *__restrict__ perm)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < K)
        perm[atomicAdd(&cursor[perm_key(reinterpret_cast<const float2 *>(mu)[k], bx_scale, by_scale, nbx, nby)], 1)] = k;
}

// stage 1: records and tile boxes, no emission
template <int C, int E>
__global__ void __launch_bounds__(PRE_NT)
k_records(int K, ParamsDev p, float R2, float sx, float sy, int oW, int oH, int nx, int ty_lo, int ty_hi,
          float *__restrict__ rec, int4 *__restrict__ tbox, HandleCtr *hc, float lscale, int mode)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < K)
        preprocess_one<C, E>(k, p, R2, sx, sy, oW, oH, nx, ty_lo, ty_hi, rec, tbox, nullptr, hc, lscale, mode);
}

// mode 2's block test from the kernel's record (mu, a, b | c at float4 0, 1)
__device__ __forceinline__ bool rec_meets(const float *rec, int rs4, int k, int tx, int ty, const BoxGeo &G, float R2)
{
    if (G.mode != 2) return true;
    const float4 f0 = reinterpret_cast<const float4 *>(rec)[(size_t)k * rs4];
    const float c = rec[(size_t)k * rs4 * 4 + 4];
    return block_meets(f0.x, f0.y, f0.z, f0.w, c, tx, ty, G, R2);
}

#ifndef SMOE_EMIT_MINB
#define SMOE_EMIT_MINB 1     // k_emit: min resident CTAs per SM (register cap; 8: config 5 -14%, config 3 +9%)
#endif
// stage 2: bucket emission, CTA-aggregated over a shared window of blocks
__global__ void __launch_bounds__(EMIT_NT, SMOE_EMIT_MINB)
k_emit(int K, const int *__restrict__ perm, const int4 *__restrict__ tbox, int nx, int ty_lo, int ty_hi,
       int *__restrict__ cnt, int *__restrict__ dids, int bcap, GridCtr *gc, double *dstats,
       const float *__restrict__ rec, int rs4, BoxGeo G, float R2)
{
    __shared__ int s_cnt[EMIT_WIN];
    __shared__ int s_base[EMIT_WIN];
    __shared__ int s_red[4][EMIT_NT / 32];
    __shared__ unsigned long long s_pairs;
    __shared__ int s_max;
    __shared__ bool last;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int i = blockIdx.x * EMIT_NT + tid;
    const int k = i < K ? __ldg(perm + i) : -1;
    SMOE_CHECK(k < K && (k >= 0 || i >= K));
    int4 tb = make_int4(0, -1, 0, -1);              // empty box
    if (k >= 0) {
        tb = tbox[k];
        if (tb.x < 0) tb = make_int4(0, -1, 0, -1);
        tb.z = max(tb.z, ty_lo);
        tb.w = min(tb.w, ty_hi - 1);
        if (tb.z > tb.w) tb = make_int4(0, -1, 0, -1);
    }
    const bool any = tb.x <= tb.y;
    // CTA window of blocks: min/max of the (non-empty) boxes
    int mnx = any ? tb.x : INT_MAX, mxx = any ? tb.y : INT_MIN, mny = any ? tb.z : INT_MAX, mxy = any ? tb.w : INT_MIN;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        mnx = min(mnx, __shfl_xor_sync(FULL, mnx, o));
        mxx = max(mxx, __shfl_xor_sync(FULL, mxx, o));
        mny = min(mny, __shfl_xor_sync(FULL, mny, o));
        mxy = max(mxy, __shfl_xor_sync(FULL, mxy, o));
    }
    if (lane == 0) { s_red[0][wid] = mnx; s_red[1][wid] = mxx; s_red[2][wid] = mny; s_red[3][wid] = mxy; }
    if (tid == 0) { s_pairs = 0ull; s_max = 0; }
    __syncthreads();
    mnx = INT_MAX; mxx = INT_MIN; mny = INT_MAX; mxy = INT_MIN;
#pragma unroll
    for (int w = 0; w < EMIT_NT / 32; w++) {
        mnx = min(mnx, s_red[0][w]); mxx = max(mxx, s_red[1][w]);
        mny = min(mny, s_red[2][w]); mxy = max(mxy, s_red[3][w]);
    }
    const int wcols = mxx - mnx + 1, wrows = mxy - mny + 1;
    const bool windowed = mxx >= mnx && (long long)wcols * wrows <= EMIT_WIN;
    const int wx = tb.y - tb.x + 1, nbx = any ? (tb.w - tb.z + 1) * wx : 0;
    int n_emit = 0, max_len = 0;
    if (windowed) {
        const int area = wcols * wrows;
        for (int w = tid; w < area; w += EMIT_NT) s_cnt[w] = 0;
        __syncthreads();
        for (int yy = tb.z; yy <= tb.w; yy++) {
            const int wrow = (yy - mny) * wcols - mnx;
            for (int xx = tb.x; xx <= tb.y; xx++) {
                if (!rec_meets(rec, rs4, k, xx, yy, G, R2)) continue;
                atomicAdd(&s_cnt[wrow + xx], 1);
                n_emit++;
            }
        }
        __syncthreads();
        // one returning global atomic per window block that has entries
        for (int w = tid; w < area; w += EMIT_NT) {
            const int c = s_cnt[w];
            if (c) {
                const int t = (mny + w / wcols) * nx + mnx + w % wcols;
                const int b = atomicAdd(&cnt[t], c);
                s_base[w] = b;
                max_len = max(max_len, b + c);
                s_cnt[w] = 0;                          // reused as the slot cursor
            }
        }
        __syncthreads();
        for (int yy = tb.z; yy <= tb.w; yy++) {
            const int wrow = (yy - mny) * wcols - mnx;
            for (int xx = tb.x; xx <= tb.y; xx++) {
                if (!rec_meets(rec, rs4, k, xx, yy, G, R2)) continue;
                const int w = wrow + xx;
                const int sl = s_base[w] + atomicAdd(&s_cnt[w], 1);
                SMOE_CHECK(w >= 0 && w < EMIT_WIN && yy >= ty_lo && yy < ty_hi && xx >= 0 && xx < nx);
                if (sl < bcap) dids[(size_t)(yy * nx + xx) * bcap + sl] = k;
            }
        }
    } else {
        // window too large (huge or scattered kernels): per-entry atomics
        int yy = tb.z, xx = tb.x;
        for (int e0 = 0; e0 < nbx; e0 += PRE_ATOM) {
            int t[PRE_ATOM], sl[PRE_ATOM];
            bool on[PRE_ATOM];
#pragma unroll
            for (int q = 0; q < PRE_ATOM; q++) {
                t[q] = yy * nx + xx;
                on[q] = e0 + q < nbx && rec_meets(rec, rs4, k, xx, yy, G, R2);
                sl[q] = on[q] ? atomicAdd(&cnt[t[q]], 1) : bcap;
                if (++xx > tb.y) { xx = tb.x; yy++; }
            }
#pragma unroll
            for (int q = 0; q < PRE_ATOM; q++) {
                if (sl[q] < bcap) dids[(size_t)t[q] * bcap + sl[q]] = k;
                if (on[q]) { max_len = max(max_len, sl[q] + 1); n_emit++; }
            }
        }
    }
    // this CTA's pairs and longest slot to the grid counters; the last CTA
    // publishes P and the overflow latch (finish_direct)
    unsigned long long pe = (unsigned)n_emit;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        pe += __shfl_xor_sync(FULL, pe, o);
        max_len = max(max_len, __shfl_xor_sync(FULL, max_len, o));
    }
    if (lane == 0) {
        if (pe) atomicAdd(&s_pairs, pe);
        if (max_len) atomicMax(&s_max, max_len);
    }
    __syncthreads();
    if (tid == 0) {
        if (s_pairs) atomicAdd(&gc->acc_pairs, s_pairs);
        if (s_max) atomicMax(&gc->acc_max, s_max);
        last = atom_add_acq_rel_gpu(&gc->ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    finish_direct(bcap, gc, dstats);
    if (tid == 0) { gc->ticket = 0; gc->work = 0; }
}

// Large grids (n_tiles > SCAN_SINGLE_MAX): single-pass decoupled look-back
// scan of the block counts, 4096 counts per CTA.  Each CTA takes a virtual
// index from a counter (so predecessors are always resident), publishes its
// aggregate, accumulates its predecessors' published values, publishes its
// inclusive prefix.  Status words carry an epoch tag so nothing needs
// clearing between scans; the last CTA to finish resets the counters.
constexpr int SCAN_SINGLE_MAX = 32768;
constexpr int LB_NT = 256, LB_IPT = 16, LB_CHUNK = LB_NT * LB_IPT;

__device__ __forceinline__ unsigned long long lb_pack(unsigned epoch, unsigned flag, long long v)
{
    return ((unsigned long long)(epoch & 0xffffffu) << 40) | ((unsigned long long)flag << 38) |
           (unsigned long long)v;
}

__global__ void __launch_bounds__(LB_NT)
k_scan_lookback(int *__restrict__ cnt, int n, int *__restrict__ start, int *__restrict__ cursor,
                long long cap, GridCtr *gc, double *dstats, unsigned long long *state)
{
    __shared__ int vid_s;
    __shared__ unsigned epoch_s;
    __shared__ int wtot[LB_NT / 32];
    __shared__ long long excl_s;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) {
        vid_s = (int)atomicAdd(&gc->scan_vid, 1u);
        epoch_s = (*(volatile unsigned *)&gc->epoch + 1u) & 0xffffffu;
    }
    __syncthreads();
    const int vid = vid_s;
    const unsigned epoch = epoch_s;
    if (vid == 0 && tid < 4 && dstats) dstats[tid] = 0.0;
    const int base = vid * LB_CHUNK + tid * LB_IPT;
    int v[LB_IPT];
    int loc = 0;
#pragma unroll
    for (int q = 0; q < LB_IPT; q++) {
        v[q] = (base + q < n) ? __ldcg(cnt + base + q) : 0;
        loc += v[q];
    }
    int inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) wtot[wid] = inc;
    __syncthreads();
    int wpre = 0, agg = 0;
#pragma unroll
    for (int w = 0; w < LB_NT / 32; w++) {
        wpre += (w < wid) ? wtot[w] : 0;
        agg += wtot[w];
    }
    if (tid == 0) {
        long long ex = 0;
        if (vid == 0) {
            atomicExch(state + vid, lb_pack(epoch, 2u, agg));
        } else {
            atomicExch(state + vid, lb_pack(epoch, 1u, agg));
            for (int j = vid - 1; j >= 0;) {
                unsigned long long sw = *(volatile unsigned long long *)(state + j);
                if ((unsigned)(sw >> 40) != epoch || ((sw >> 38) & 3u) == 0u) continue;   // not yet published
                ex += (long long)(sw & ((1ull << 38) - 1));
                if (((sw >> 38) & 3u) == 2u) break;
                j--;
            }
            atomicExch(state + vid, lb_pack(epoch, 2u, ex + agg));
        }
        excl_s = ex;
    }
    __syncthreads();
    int e = (int)excl_s + wpre + inc - loc;
#pragma unroll
    for (int q = 0; q < LB_IPT; q++) {
        if (base + q < n) {
            start[base + q] = e;
            cursor[base + q] = e;
            cnt[base + q] = 0;
        }
        e += v[q];
    }
    const int nblk = (n + LB_CHUNK - 1) / LB_CHUNK;
    if (tid == 0 && vid == nblk - 1) {
        long long P = excl_s + agg;
        start[n] = (int)P;
        gc->pairs = P;
        gc->skip = P > cap ? 1u : 0u;
        if (P > cap) {
            if (P > gc->need) gc->need = P;
            gc->skipped += 1;
        }
    }
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(&gc->scan_done, 1u) == (unsigned)nblk - 1) {
            gc->scan_vid = 0;
            gc->scan_done = 0;
            gc->epoch = epoch;
            __threadfence();
        }
    }
}

// ---------------------------------------------------------------- a3 ------
// First radix digit: every block b_n inside kernel k's box records k
// ("Each intersected block b_n is recorded").
__global__ void __launch_bounds__(64)
k_scatter(int K, const int4 *__restrict__ tbox, int nx, int ty_lo, int ty_hi,
          int *__restrict__ cursor, int *__restrict__ ids, long long cap, const GridCtr *gc,
          const float *__restrict__ rec, int rs4, BoxGeo G, float R2)
{
    if (gc->skip) return;
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    int4 tb = tbox[k];
    if (tb.x < 0) return;
    int y0 = max(tb.z, ty_lo), y1 = min(tb.w, ty_hi - 1);
    if (y0 > y1) return;
    const int w = tb.y - tb.x + 1, cnt = w * (y1 - y0 + 1);
    // issue the bucket atomics in groups of 8 so their latencies overlap
    for (int i0 = 0; i0 < cnt; i0 += 8) {
        int pos[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            int i = i0 + q;
            pos[q] = -1;
            if (i < cnt) {
                int tyy = y0 + i / w, txx = tb.x + i % w;
                if (rec_meets(rec, rs4, k, txx, tyy, G, R2)) pos[q] = atomicAdd(&cursor[tyy * nx + txx], 1);
            }
        }
#pragma unroll
        for (int q = 0; q < 8; q++)
            if (pos[q] >= 0) ids[pos[q]] = k;
    }
}

// ------------------------------------------------- a1-a4 fused (default) --
// One cooperative launch bins a grid: phase 1 preprocesses the kernels and
// counts (grid-stride, = k_preprocess); phase 2 scans the block counts in
// parallel (every CTA owns a contiguous chunk of blocks: chunk totals, grid
// sync, chunk offsets by a CTA-level sum, local scan) and histograms the
// list lengths for the LPT order; phase 3 scatters the kernel ids into their
// buckets (= k_scatter) and writes the LPT block order.  Three grid-wide
// barriers replace two kernel boundaries and the serial last-CTA scan.
struct BinArgs {
    int K;
    ParamsDev p;
    float R2, sx, sy, lscale;
    int oW, oH, nx, ty_lo, ty_hi, n_tiles;
    float *rec;
    int4 *tbox;
    int *cnt, *start, *cursor, *ids, *order;
    int *chunk;          // [gridDim] chunk totals
    int *hist;           // [512]: LPT bin counts | bin cursors
    long long cap;
    GridCtr *gc;
    HandleCtr *hc;
    double *dstats;
    int mode, rs4;
};

constexpr int BIN_NT = 256;

template <int C, int E>
__global__ void __launch_bounds__(BIN_NT)
k_bin(BinArgs B)
{
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nthreads = gridDim.x * BIN_NT;
    __shared__ int sw[BIN_NT / 32];
    __shared__ long long s_off;
    __shared__ int shist[256];
    // ---- phase 1 (a1) ----
    if (blockIdx.x == 0) {
        for (int i = tid; i < 512; i += BIN_NT) B.hist[i] = 0;
        if (tid < 4 && B.dstats) B.dstats[tid] = 0.0;
    }
    for (int k = blockIdx.x * BIN_NT + tid; k < B.K; k += nthreads)
        preprocess_one<C, E>(k, B.p, B.R2, B.sx, B.sy, B.oW, B.oH, B.nx, B.ty_lo, B.ty_hi, B.rec, B.tbox,
                             B.cnt, B.hc, B.lscale, B.mode);
    grid.sync();
    // ---- phase 2 (a2): chunked scan of the block counts ----
    const int n = B.n_tiles;
    const int ch = (n + gridDim.x - 1) / gridDim.x;
    const int c0 = min(n, blockIdx.x * ch), c1 = min(n, c0 + ch);
    int part = 0;
    for (int i = c0 + tid; i < c1; i += BIN_NT) part += __ldcg(B.cnt + i);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) part += __shfl_xor_sync(FULL, part, o);
    if (lane == 0) sw[wid] = part;
    __syncthreads();
    if (tid == 0) {
        int t = 0;
        for (int w = 0; w < BIN_NT / 32; w++) t += sw[w];
        B.chunk[blockIdx.x] = t;
    }
    shist[tid] = 0;
    grid.sync();
    {
        long long off = 0;
        for (int b = tid; b < (int)blockIdx.x; b += BIN_NT) off += __ldcg(B.chunk + b);
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) off += __shfl_xor_sync(FULL, off, o);
        __syncthreads();
        if (lane == 0) sw[wid] = (int)off;
        __syncthreads();
        if (tid == 0) {
            long long t = 0;
            for (int w = 0; w < BIN_NT / 32; w++) t += sw[w];
            s_off = t;
        }
        __syncthreads();
    }
    const int t0 = B.ty_lo * B.nx, t1 = B.ty_hi * B.nx;
    long long carry = s_off;
    for (int base = c0; base < c1; base += BIN_NT) {
        const int i = base + tid;
        const int v = i < c1 ? __ldcg(B.cnt + i) : 0;
        int inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += t;
        }
        __syncthreads();
        if (lane == 31) sw[wid] = inc;
        __syncthreads();
        int wpre = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < BIN_NT / 32; w++) {
            wpre += (w < wid) ? sw[w] : 0;
            tot += sw[w];
        }
        if (i < c1) {
            const int ex = (int)carry + wpre + inc - v;
            B.start[i] = ex;
            B.cursor[i] = ex;
            B.cnt[i] = 0;
            if (B.order && i >= t0 && i < t1) atomicAdd(&shist[255 - min(v, 255)], 1);
        }
        carry += tot;
    }
    __syncthreads();
    if (B.order && shist[tid]) atomicAdd(&B.hist[tid], shist[tid]);
    if (blockIdx.x == gridDim.x - 1 && tid == 0) {
        const long long P = carry;
        B.start[n] = (int)P;
        B.gc->pairs = P;
        B.gc->skip = P > B.cap ? 1u : 0u;
        if (P > B.cap) {
            if (P > B.gc->need) B.gc->need = P;
            B.gc->skipped += 1;
        }
    }
    grid.sync();
    // ---- phase 3 (a3 + LPT order) ----
    const long long P = __ldcg(&B.gc->pairs);
    if (P > B.cap) return;                  // uniform: every CTA reads the same P
    const BoxGeo G{B.mode, 1.0f / B.sx, 1.0f / B.sy, B.oW, B.oH};
    for (int k = blockIdx.x * BIN_NT + tid; k < B.K; k += nthreads) {
        int4 tb = B.tbox[k];
        if (tb.x < 0) continue;
        int y0 = max(tb.z, B.ty_lo), y1 = min(tb.w, B.ty_hi - 1);
        if (y0 > y1) continue;
        const int w = tb.y - tb.x + 1, cnt = w * (y1 - y0 + 1);
        for (int i0 = 0; i0 < cnt; i0 += 8) {
            int pos[8];
#pragma unroll
            for (int q = 0; q < 8; q++) {
                int i = i0 + q;
                pos[q] = -1;
                if (i < cnt && rec_meets(B.rec, B.rs4, k, tb.x + i % w, y0 + i / w, G, B.R2))
                    pos[q] = atomicAdd(&B.cursor[(y0 + i / w) * B.nx + tb.x + i % w], 1);
            }
#pragma unroll
            for (int q = 0; q < 8; q++)
                if (pos[q] >= 0) B.ids[pos[q]] = k;
        }
    }
    if (B.order) {
        // bin bases: exclusive scan of the 256 LPT bins (redundantly per CTA)
        int v = __ldcg(B.hist + tid), inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) sw[wid] = inc;
        __syncthreads();
        int wpre = 0;
        for (int w = 0; w < wid; w++) wpre += sw[w];
        shist[tid] = wpre + inc - v;
        __syncthreads();
        for (int i = max(c0, t0) + tid; i < min(c1, t1); i += BIN_NT) {
            const int c = __ldcg(B.start + i + 1) - __ldcg(B.start + i);
            const int bin = 255 - min(c, 255);
            B.order[shist[bin] + atomicAdd(&B.hist[256 + bin], 1)] = i;
        }
    }
    if (blockIdx.x == 0 && tid == 0) { B.gc->ticket = 0; B.gc->work = 0; }
}

// ---------------------------------------------------------------- a4 ------
// Second radix digit: sort each bucket by kernel id.  Buckets up to SORT_CAP
// are bitonic-sorted in shared memory; larger ones are sorted in SORT_CAP
// runs and merged in global memory (ids are unique, so the merge position of
// an element is its index plus its rank in the other run).
__device__ __forceinline__ void smem_bitonic(int *s, int np)
{
    for (int k = 2; k <= np; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < np; i += blockDim.x) {
                int ixj = i ^ j;
                if (ixj > i) {
                    int a = s[i], b = s[ixj];
                    bool asc = (i & k) == 0;
                    if ((a > b) == asc) { s[i] = b; s[ixj] = a; }
                }
            }
            __syncthreads();
        }
}

__device__ __forceinline__ int lower_bound_i(const int *a, int n, int x)
{
    int lo = 0, hi = n;
    while (lo < hi) {
        int m = (lo + hi) >> 1;
        if (a[m] < x) lo = m + 1; else hi = m;
    }
    return lo;
}

// Warp-level bitonic sort of up to 32*R ints held in registers, element
// e = i*32 + lane (coalesced loads/stores).  Stages with partner distance
// j < 32 exchange through shuffles, j >= 32 swap registers of one lane.
template <int R>
__device__ __forceinline__ void warp_bitonic(int (&v)[R], int lane)
{
#pragma unroll
    for (int k = 2; k <= 32 * R; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < 32) {
#pragma unroll
                for (int i = 0; i < R; i++) {
                    int e = i * 32 + lane;
                    int o = __shfl_xor_sync(FULL, v[i], j);
                    bool asc = (e & k) == 0, lower = (lane & j) == 0;
                    v[i] = (lower == asc) ? min(v[i], o) : max(v[i], o);
                }
            } else {
#pragma unroll
                for (int i = 0; i < R; i++) {
                    int ii = i ^ (j >> 5);
                    if (ii > i) {
                        int e = i * 32 + lane;
                        bool asc = (e & k) == 0;
                        int a = v[i], b = v[ii];
                        v[i] = asc ? min(a, b) : max(a, b);
                        v[ii] = asc ? max(a, b) : min(a, b);
                    }
                }
            }
        }
    }
}

template <int R>
__device__ __forceinline__ void warp_sort_seg(int *seg, int n, int lane)
{
    int v[R];
#pragma unroll
    for (int i = 0; i < R; i++) v[i] = (i * 32 + lane < n) ? seg[i * 32 + lane] : 0x7fffffff;
    warp_bitonic<R>(v, lane);
#pragma unroll
    for (int i = 0; i < R; i++)
        if (i * 32 + lane < n) seg[i * 32 + lane] = v[i];
}

// Sort one bucket of n kernel ids in place with the whole CTA: chunks of
// `chunk` (a power of two fitting the shared buffer s) are bitonic-sorted in
// shared memory, then merged pairwise through global scratch `tmp` (ids are
// unique, so an element's merged position is its index plus its rank in the
// other run).
__device__ __noinline__ void cta_sort_seg(int *seg, int n, int *tmp, int *s, int chunk)
{
    for (int c0 = 0; c0 < n; c0 += chunk) {
        int m = min(chunk, n - c0);
        int np = 32;
        while (np < m) np <<= 1;
        __syncthreads();
        for (int i = threadIdx.x; i < np; i += blockDim.x) s[i] = i < m ? seg[c0 + i] : 0x7fffffff;
        __syncthreads();
        smem_bitonic(s, np);
        for (int i = threadIdx.x; i < m; i += blockDim.x) seg[c0 + i] = s[i];
    }
    __syncthreads();
    if (n <= chunk) return;
    int *src = seg, *dst = tmp;
    for (int run = chunk; run < n; run <<= 1) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            int lo = (i / (2 * run)) * (2 * run);
            int mid = min(lo + run, n), hi = min(lo + 2 * run, n);
            int x = src[i];
            int pos;
            if (i < mid) pos = (i - lo) + lower_bound_i(src + mid, hi - mid, x);
            else pos = (i - mid) + lower_bound_i(src + lo, mid - lo, x);
            dst[lo + pos] = x;
        }
        __syncthreads();
        int *sw = src; src = dst; dst = sw;
    }
    if (src != seg)
        for (int i = threadIdx.x; i < n; i += blockDim.x) seg[i] = src[i];
    __syncthreads();
}

// Second radix digit of the binning, run at the start of every raster CTA
// on its own bucket: <= 256 ids are sorted by warp 0 in registers, larger
// buckets by the whole CTA.  The sorted bucket is written back, so the global
// list is the canonical (block, kernel) order that smoe_bin reports.
__device__ __forceinline__ void sort_bucket(int *seg, int n, int *tmp, int *s, int chunk)
{
    if (n <= 1) return;
    if (n <= 256) {
        // one warp in registers while the other three wait at the next
        // barrier (a four-warp version -- quarter runs + rank merge by binary
        // search -- measured 3% slower at configs 2-4: DESIGN.md §10)
        if (threadIdx.x < 32) {
            int lane = threadIdx.x;
            if (n <= 32) warp_sort_seg<1>(seg, n, lane);
            else if (n <= 64) warp_sort_seg<2>(seg, n, lane);
            else if (n <= 128) warp_sort_seg<4>(seg, n, lane);
            else warp_sort_seg<8>(seg, n, lane);
        }
        return;   // the caller's next __syncthreads publishes the result
    }
    cta_sort_seg(seg, n, tmp, s, chunk);
}

// ------------------------------------------------------- a5 / a6 / a7 -----
struct RasterArgs {
    const int *order;     // LPT block order (k_preprocess)
    GridCtr *gcw;         // work-queue head
    int n_work;           // number of blocks in the order
    int n_sm;             // SM count (stratum width of the LPT assignment)
    const float *rec;
    int *ids;             // block lists (bucket-sorted in place by the raster)
    int *tmp;             // merge scratch for buckets larger than the smem chunk
    const int *start;     // CSR lists: block t = ids[start[t], start[t+1])
    int *len;             // direct buckets (len != null): block t = ids[t bcap, t bcap + len[t]);
                          // len = the binning's count array, reset by the block's CTA
    int *lenout;          // direct buckets: copy of len for the diagnostics (smoe_bin)
    int K;                // pool size (debug bounds checks)
    int bcap;
    const GridCtr *gc;
    long long cap;
    int nx, tile0;
    int oW, oH;
    float sx, sy;        // source spacing of output samples: x = (j+1/2) sx - 1/2
    float R2;
    int rbf;              // 1: RBF head y = sum_j m_j(x) pi_j K_j (Eq. 1), no gate normalisation
    // training
    const float *target; // [C][H][W] (H = oH, W = oW in training)
    float e_scale;        // 2 / (H W C): dL/dy = e_scale (y - t)
    float *acc;           // raw per-kernel sums [K][V]
    double *dstats;       // SSE, clamped SSE, uncovered pixels
    // render
    float *out;           // [C][oH][oW]
    float accum;          // 0: out = y; else out += accum * y
    int vec_out;          // 1: float4 row stores through shared memory
    // profiling (PROF instantiation only): tested / hit (pixel, kernel)
    // pairs, SM cycles in the bucket sort, SM cycles of the whole CTA
    unsigned long long *work;
};

// Multi-value warp reduction ("transpose" butterfly): V values per lane ->
// lane holds the warp total of value idx(lane).  log2(V) exchange steps move
// half of the remaining values each, then plain butterflies finish.
template <int V>
__device__ __forceinline__ float warp_reduce_transpose(float (&v)[V], int lane, int &idx)
{
    idx = 0;
#pragma unroll
    for (int n = V, off = 16; n > 1; n >>= 1, off >>= 1) {
        bool up = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < n / 2; i++) {
            float send = up ? v[i] : v[i + n / 2];
            float keep = up ? v[i + n / 2] : v[i];
            v[i] = keep + __shfl_xor_sync(FULL, send, off);
        }
        if (up) idx += n / 2;
    }
    constexpr int LOGV = V == 8 ? 3 : (V == 16 ? 4 : (V == 4 ? 2 : (V == 2 ? 1 : 5)));
#pragma unroll
    for (int off = 16 >> LOGV; off >= 1; off >>= 1) v[0] += __shfl_xor_sync(FULL, v[0], off);
    return v[0];
}

// One CTA = one 16x16 block b_n, 128 threads = 4 warps, each warp an 8x8
// quadrant, each lane a vertical pair of pixels.  The block's kernel list
// K_n is staged through shared memory in batches of BATCH; a warp skips a
// kernel when none of its 64 pixels is inside the kernel's ellipse
// (warp-uniform branch).
//
// Forward (a5): D = sum g, N_c = sum g m_c(x) per pixel in registers.
// RENDER: y = N/D written to out.  TRAIN: loss partials (a6), then the
// backward (a7) in one of two forms:
//   KPAR = false  pixel-parallel (default): every warp re-sweeps K_n, per (warp,
//                 kernel) the raw gradient sums are reduced across the warp
//                 (transpose butterfly) and added with one atomic per value.
//   KPAR = true   kernel-parallel: the forward records, per kernel, the
//                 256-bit mask of block pixels inside its ellipse; per-pixel
//                 backward seeds go to shared memory; then groups of L lanes
//                 own one kernel each (heaviest first, so lanes of a warp
//                 carry similar pixel counts) and walk only its masked pixels,
//                 accumulating the raw sums in registers -- no per-pixel
//                 reduction, one vector of atomics per kernel and block.
// Mask bit layout: word 2w+h (warp w, h = upper/lower pixel of the lane's
// pair), bit l = lane l: col = (w&1)*8 + (l&7), row = (w>>1)*8 + (l>>3)*2 + h.
template <int C, int E, bool TRAIN, bool PROF, bool KPAR>
__device__ __forceinline__ void raster_tile(const RasterArgs &A, const int tile)
{
    using R = Rec<C, E>;
    constexpr int RS4 = R::RS / 4;
    constexpr int BATCH = SMOE_RASTER_BATCH;
    // forward kernel-loop unroll: 4 for constant experts (+2% at config 3);
    // linear ones: 2 in the kernel-parallel train raster (+2% at config 2),
    // none in the 40-register forms (spills)
    constexpr bool MASKS = TRAIN && KPAR;
    constexpr int FWD_UNROLL = (E == 3) ? (MASKS ? 2 : 1) * kFwdUnroll : 4 * kFwdUnroll;
    __shared__ float4 srec[BATCH * RS4];
    __shared__ int sid[BATCH];
    // per-lane backward seeds of the lane's pixel pair, packed by pixel:
    // [warp][lane] = C = 1: {(eD_0, eD_0'), (K, K')}, {(x, y0), -}
    //                C = 3: {(eD_0, eD_0'), (eD_1, eD_1')}, {(eD_2, eD_2'), (K, K')}, {(x, y0), -}
    // with (x, y0) the lane's upper pixel in source coordinates
    constexpr int NSEED = C == 1 ? 2 : 3;
    __shared__ float4 spix[MASKS ? 128 * NSEED : 1];
    // per-warp kernel records of the pair list: {upper-pixel ballot, lower-pixel
    // ballot, kernel slot in the batch, entries before it}; a lane with either
    // pixel inside is one entry (a vertical pixel pair)
    __shared__ uint4 skr[MASKS ? 4 : 1][MASKS ? BATCH : 1];
    __shared__ double red[3][4];

    const int tx = tile % A.nx, ty = tile / A.nx;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int px = tx * TILE + (warp & 1) * 8 + (lane & 7);
    const int py0 = ty * TILE + (warp >> 1) * 8 + (lane >> 3) * 2, py1 = py0 + 1;
    const bool v0 = px < A.oW && py0 < A.oH, v1 = px < A.oW && py1 < A.oH;
    // XF (render, constant experts; SMOE_R4_XF): the block-centred records
    // of k_render4 -- coordinates relative to the block's first sample, the
    // staged record's first float4 rewritten to {a, -a mx, b, -(b mx + c my)}
    // -- so the cull test is FFMA, FFMA, FFMA2 + FMUL, FFMA2.  (The train
    // raster measured slower with it: DESIGN.md §10.)
    constexpr bool XF = SMOE_R4_XF && !TRAIN && E == 1 && C == 3;   // (C = 1 spills at the 40-register bound)
    const float X0 = XF ? (tx * TILE + 0.5f) * A.sx - 0.5f : 0.f;
    const float Y0 = XF ? (ty * TILE + 0.5f) * A.sy - 0.5f : 0.f;
    const float xs = (px + 0.5f) * A.sx - 0.5f - X0;
    const float ys0 = (py0 + 0.5f) * A.sy - 0.5f - Y0, ys1 = (py1 + 0.5f) * A.sy - 0.5f - Y0;
    const float R2 = A.R2;
    const int s0 = A.len ? tile * A.bcap : A.start[tile];
    const int n = A.len ? A.len[tile] : A.start[tile + 1] - s0;
    // direct buckets: the count is consumed here and reset for the next
    // binning (when n > 0 every thread has read it before thread 0 passes the
    // first batch barrier, and thread 0 resets it only at its return)
    // PROF: SM cycles of this CTA in the bucket sort (a4) and in total
    const long long c_start = PROF ? clock64() : 0;
    auto release = [&] {
        if (A.len && threadIdx.x == 0) {
            A.lenout[tile] = n;
            if (n) A.len[tile] = 0;
        }
        if (PROF && threadIdx.x == 0) atomicAdd(&A.work[3], (unsigned long long)(clock64() - c_start));
    };
    // a4 (second digit): sort this block's bucket by kernel id; srec doubles
    // as the shared scratch (its capacity in ints is a power of two >= 1024)
    constexpr int SCHUNK = (BATCH * RS4 * 4 >= 2048) ? 2048 : 1024;
    sort_bucket(A.ids + s0, n, A.tmp + s0, reinterpret_cast<int *>(srec), SCHUNK);
    if (PROF) {
        __syncthreads();
        if (threadIdx.x == 0) atomicAdd(&A.work[2], (unsigned long long)(clock64() - c_start));
    }

    float2 D2 = make_float2(0.f, 0.f), N2[C];
#pragma unroll
    for (int c = 0; c < C; c++) N2[c] = make_float2(0.f, 0.f);
    unsigned long long w_tested = 0, w_hit = 0;
    int wrun = 0, nrec = 0;                        // entries / kernel records this warp listed (KPAR)
    const int w_valid = PROF ? __popc(__ballot_sync(FULL, v0)) + __popc(__ballot_sync(FULL, v1)) : 0;

    auto load_batch = [&](int b0, int nb) {
        __syncthreads();
        for (int i = threadIdx.x; i < nb * RS4; i += blockDim.x) {
            int j = i / RS4, q = i - j * RS4;
            int id = A.ids[s0 + b0 + j];
            SMOE_CHECK(id >= 0 && id < A.K && (A.len ? b0 + j < A.bcap : s0 + b0 + j < A.cap));
            srec[i] = reinterpret_cast<const float4 *>(A.rec)[(size_t)id * RS4 + q];
            if (TRAIN && q == 0) sid[j] = id;
        }
        __syncthreads();
        if (XF) {
            for (int j = threadIdx.x; j < nb; j += blockDim.x) {
                const float4 f0 = srec[j * RS4];
                const float c = srec[j * RS4 + 1].x;
                const float mx = f0.x - X0, my = f0.y - Y0;
                srec[j * RS4] = make_float4(f0.z, -f0.z * mx, f0.w, -fmaf(f0.w, mx, c * my));
            }
            __syncthreads();
        }
    };
    auto load_rec = [&](int j, float (&r)[R::RS]) {
#pragma unroll
        for (int q = 0; q < RS4; q++) {
            float4 f = srec[j * RS4 + q];
            r[4 * q] = f.x; r[4 * q + 1] = f.y; r[4 * q + 2] = f.z; r[4 * q + 3] = f.w;
        }
    };
    // d^2 of this lane's two pixels for record r
    // The lane's two pixels share dx and differ in dy: their arithmetic is
    // done pairwise with packed f32x2 instructions (FADD2/FMUL2/FFMA2, sm_100).
    const float2 ys2 = make_float2(ys0, ys1);
    auto dist2 = [&](const float (&r)[R::RS], float &dx, float2 &dy, float &u, float2 &w, float2 &q) {
        if (XF) {   // dx, dy unused (constant experts, no backward)
            dx = 0.f;
            dy = make_float2(0.f, 0.f);
            u = fmaf(r[0], xs, r[1]);
            const float bx = fmaf(r[2], xs, r[3]);
            w = __ffma2_rn(make_float2(r[4], r[4]), ys2, make_float2(bx, bx));
        } else {
            dx = xs - r[0];
            dy = __fadd2_rn(ys2, make_float2(-r[1], -r[1]));
            u = r[2] * dx;
            const float bdx = r[3] * dx;
            w = __ffma2_rn(make_float2(r[4], r[4]), dy, make_float2(bdx, bdx));
        }
        const float uu = u * u;
        q = __ffma2_rn(w, w, make_float2(uu, uu));
    };

    // ---- forward (Eq. 5 with the per-pixel cull of P:221) ----
    // LIST: also append this warp's list entries (kernel-parallel backward,
    // K_n within one batch); a separate instantiation keeps the test out of
    // the kernel loop
    auto forward = [&](auto list_tag) {
        constexpr bool LIST = decltype(list_tag)::value;
        for (int b0 = 0; b0 < n; b0 += BATCH) {
            int nb = min(BATCH, n - b0);
            load_batch(b0, nb);
            // software pipeline: the test half of record j+1 (mu, a, b, c and
            // the next four floats) is loaded while record j is tested
            float4 n0 = srec[0], n1 = srec[1];
#pragma unroll FWD_UNROLL
            for (int j = 0; j < nb; j++) {
                float r[R::RS];
                if (SMOE_FWD_PREFETCH) {
                    const float4 f0 = n0, f1 = n1;
                    if (j + 1 < nb) { n0 = srec[(j + 1) * RS4]; n1 = srec[(j + 1) * RS4 + 1]; }
                    r[0] = f0.x; r[1] = f0.y; r[2] = f0.z; r[3] = f0.w;
                    r[4] = f1.x; r[5] = f1.y; r[6] = f1.z; r[7] = f1.w;
#pragma unroll
                    for (int q4 = 2; q4 < RS4; q4++) {
                        const float4 f = srec[j * RS4 + q4];
                        r[4 * q4] = f.x; r[4 * q4 + 1] = f.y; r[4 * q4 + 2] = f.z; r[4 * q4 + 3] = f.w;
                    }
                } else {
                    load_rec(j, r);
                }
                float dx, u;
                float2 dy, w, q;
                dist2(r, dx, dy, u, w, q);
                bool h0 = v0 && q.x <= R2, h1 = v1 && q.y <= R2;
                unsigned b0m = __ballot_sync(FULL, h0), b1m = __ballot_sync(FULL, h1);
                if (PROF) {
                    w_tested += w_valid;
                    w_hit += __popc(b0m) + __popc(b1m);
                }
                if ((b0m | b1m) == 0u) continue;
                if (LIST) {
                    // one record per (warp, kernel) with a hit: its two
                    // ballots and the entries listed before it
                    if (lane == 0) skr[warp][nrec] = make_uint4(b0m, b1m, (unsigned)j, (unsigned)wrun);
                    nrec++;
                    wrun += __popc(b0m | b1m);
                }
                const float2 ea = __ffma2_rn(q, make_float2(-0.5f * LOG2E, -0.5f * LOG2E), make_float2(r[5], r[5]));
                const float2 g = make_float2(h0 ? ex2_approx(ea.x) : 0.f, h1 ? ex2_approx(ea.y) : 0.f);
                D2 = __fadd2_rn(D2, g);
#pragma unroll
                for (int c = 0; c < C; c++) {
                    float2 m = make_float2(r[6 + c * E], r[6 + c * E]);
                    if (E == 3) {
                        const float mb = fmaf(r[6 + c * E + 1], dx, r[6 + c * E]);
                        m = __ffma2_rn(make_float2(r[6 + c * E + 2], r[6 + c * E + 2]), dy, make_float2(mb, mb));
                    }
                    N2[c] = __ffma2_rn(g, m, N2[c]);
                }
            }
        }
    };
    if (MASKS && n <= BATCH) forward(std::true_type{});
    else forward(std::false_type{});
    if (PROF && lane == 0) {
        atomicAdd(&A.work[0], w_tested);
        atomicAdd(&A.work[1], w_hit);
    }
    const float D0 = D2.x, D1 = D2.y;
    float y0[C], y1[C];
    // SMoE (Eq. 2/4): y = N/D.  RBF head (Eq. 1): y = N, i.e. "D" = 1.
    float iD0 = A.rbf ? 1.f : (D0 > 0.f ? 1.0f / D0 : 0.f), iD1 = A.rbf ? 1.f : (D1 > 0.f ? 1.0f / D1 : 0.f);
#pragma unroll
    for (int c = 0; c < C; c++) { y0[c] = N2[c].x * iD0; y1[c] = N2[c].y * iD1; }

    if (!TRAIN && !A.vec_out) {
        // scalar epilogue (default): each lane stores its two pixels per
        // channel; a warp store covers 4 rows x 32 contiguous bytes (full
        // sectors).  Measured 1.7% faster than the float4 epilogue below at
        // the config-3 4x render (the staging costs more issue slots than
        // the 4x fewer stores save; the render is not store-bound).
        size_t plane = (size_t)A.oH * A.oW;
        float *o0 = A.out + (size_t)py0 * A.oW + px, *o1 = A.out + (size_t)py1 * A.oW + px;
#pragma unroll
        for (int c = 0; c < C; c++) {
            if (A.accum != 0.f) {
                if (v0) o0[c * plane] = fmaf(A.accum, y0[c], o0[c * plane]);
                if (v1) o1[c * plane] = fmaf(A.accum, y1[c], o1[c * plane]);
            } else {
                if (v0) o0[c * plane] = y0[c];
                if (v1) o1[c * plane] = y1[c];
            }
        }
        release();
        return;
    }
    if (!TRAIN) {
        // Render epilogue: the block's C x 16 x 16 outputs are staged in
        // shared memory and written as
        // coalesced float4 rows (st.global.v4: 16 B per thread, a block row is
        // one 64-byte run).  Row stride 20 floats keeps the lane-pair layout
        // of the staging writes free of bank conflicts and every float4
        // 16-byte aligned.  Ragged edges and rasters whose width is not a
        // multiple of 4 store the remaining pixels one by one.
        constexpr int SR = 20;
        __shared__ float so[TRAIN ? 1 : C * TILE * SR];   // own buffer: no barrier before the staging writes
        const int cx = (warp & 1) * 8 + (lane & 7), cy = (warp >> 1) * 8 + (lane >> 3) * 2;
#pragma unroll
        for (int c = 0; c < C; c++) {
            so[(c * TILE + cy) * SR + cx] = y0[c];
            so[(c * TILE + cy + 1) * SR + cx] = y1[c];
        }
        __syncthreads();
        const size_t plane = (size_t)A.oH * A.oW;
        const bool vec = ((A.oW & 3) == 0) && ((reinterpret_cast<uintptr_t>(A.out) & 15) == 0);
        const int x0 = tx * TILE, y0r = ty * TILE;
        for (int i = threadIdx.x; i < C * TILE * 4; i += blockDim.x) {
            const int c = i / (TILE * 4), r = (i >> 2) & (TILE - 1), q = i & 3;
            const int y = y0r + r, x = x0 + 4 * q;
            if (y >= A.oH || x >= A.oW) continue;
            const float4 v = *reinterpret_cast<const float4 *>(so + (c * TILE + r) * SR + 4 * q);
            float *o = A.out + c * plane + (size_t)y * A.oW + x;
            if (vec && x + 3 < A.oW) {
                float4 *o4 = reinterpret_cast<float4 *>(o);
                if (A.accum != 0.f) {          // multi-model fusion: out += w y (Eq. 11)
                    float4 a = *o4;
                    a.x = fmaf(A.accum, v.x, a.x); a.y = fmaf(A.accum, v.y, a.y);
                    a.z = fmaf(A.accum, v.z, a.z); a.w = fmaf(A.accum, v.w, a.w);
                    *o4 = a;
                } else {
                    *o4 = v;
                }
            } else {
                const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int e = 0; e < 4; e++)
                    if (x + e < A.oW) o[e] = A.accum != 0.f ? fmaf(A.accum, vv[e], o[e]) : vv[e];
            }
        }
        release();
        return;
    }

    // ---- loss / PSNR partials (Q8) and per-pixel backward seeds ----
    // eD_c = (dL/dy_c) / D and K = sum_c eD_c y_c, so that for a kernel
    // inside the ellipse G = sum_c eD_c m_c(x) - K and s = dL/d(d^2) = -g G / 2.
    float eD0[C], eD1[C], K0 = 0.f, K1 = 0.f;
    {
        // lane and warp partials in fp32 (<= 192 terms), block and image sums in fp64
        float sse = 0.f, ssec = 0.f, unc = 0.f;
        size_t plane = (size_t)A.oH * A.oW;
#pragma unroll
        for (int c = 0; c < C; c++) {
            float t0 = v0 ? A.target[c * plane + (size_t)py0 * A.oW + px] : 0.f;
            float t1 = v1 ? A.target[c * plane + (size_t)py1 * A.oW + px] : 0.f;
            float r0 = v0 ? y0[c] - t0 : 0.f, r1 = v1 ? y1[c] - t1 : 0.f;
            float rc0 = v0 ? __saturatef(y0[c]) - __saturatef(t0) : 0.f;
            float rc1 = v1 ? __saturatef(y1[c]) - __saturatef(t1) : 0.f;
            sse = fmaf(r0, r0, fmaf(r1, r1, sse));
            ssec = fmaf(rc0, rc0, fmaf(rc1, rc1, ssec));
            eD0[c] = A.e_scale * r0 * iD0;      // 0 if uncovered
            eD1[c] = A.e_scale * r1 * iD1;
            if (!A.rbf) {                       // RBF: dy/dg = m(x), no -y term
                K0 = fmaf(eD0[c], y0[c], K0);
                K1 = fmaf(eD1[c], y1[c], K1);
            }
        }
        unc = (float)(((v0 && D0 <= 0.f) ? 1 : 0) + ((v1 && D1 <= 0.f) ? 1 : 0));
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            sse += __shfl_xor_sync(FULL, sse, o);
            ssec += __shfl_xor_sync(FULL, ssec, o);
            unc += __shfl_xor_sync(FULL, unc, o);
        }
        if (lane == 0) { red[0][warp] = (double)sse; red[1][warp] = (double)ssec; red[2][warp] = (double)unc; }
        if (MASKS) {
            if (SMOE_SEED_SOA) {
                // one float per (component, thread): component k of thread t at
                // [k * 128 + t] -- the backward's 32-bit loads of random pixel
                // slots hit 32 distinct banks (no conflicts; more loads)
                float *sf = reinterpret_cast<float *>(spix) + threadIdx.x;
                if (C == 1) {
                    sf[0] = eD0[0]; sf[128] = eD1[0]; sf[256] = K0; sf[384] = K1; sf[512] = xs; sf[640] = ys0;
                } else {
#pragma unroll
                    for (int c = 0; c < C; c++) { sf[256 * c] = eD0[c]; sf[256 * c + 128] = eD1[c]; }
                    sf[256 * C] = K0; sf[256 * C + 128] = K1; sf[256 * C + 256] = xs; sf[256 * C + 384] = ys0;
                }
            } else {
            float4 *sp = spix + NSEED * threadIdx.x;
            if (C == 1) {
                sp[0] = make_float4(eD0[0], eD1[0], K0, K1);
                sp[1] = make_float4(xs, ys0, 0.f, 0.f);
            } else {
                sp[0] = make_float4(eD0[0], eD1[0], eD0[C > 1 ? 1 : 0], eD1[C > 1 ? 1 : 0]);
                sp[1] = make_float4(eD0[C > 2 ? 2 : 0], eD1[C > 2 ? 2 : 0], K0, K1);
                sp[2] = make_float4(xs, ys0, 0.f, 0.f);
            }
            }
        }
        __syncthreads();
        if (threadIdx.x < 3) {
            double sm = red[threadIdx.x][0] + red[threadIdx.x][1] + red[threadIdx.x][2] + red[threadIdx.x][3];
            if (sm != 0.0) atomicAdd(&A.dstats[threadIdx.x], sm);
        }
    }

    if (!KPAR) {
        // ---- pixel-parallel backward (raw sums per kernel) ----
        for (int b0 = 0; b0 < n; b0 += BATCH) {
            int nb = min(BATCH, n - b0);
            if (n > BATCH) load_batch(b0, nb);   // n <= BATCH: batch 0 is still resident
            for (int j = 0; j < nb; j++) {
                float r[R::RS];
                load_rec(j, r);
                float dx, u;
                float2 dyv, wv, qv;
                dist2(r, dx, dyv, u, wv, qv);
                const float dy0 = dyv.x, dy1 = dyv.y, w0 = wv.x, w1 = wv.y, q0 = qv.x, q1 = qv.y;
                bool h0 = v0 && q0 <= R2 && D0 > 0.f, h1 = v1 && q1 <= R2 && D1 > 0.f;
                if (!__any_sync(FULL, h0 || h1)) continue;
                float g0 = h0 ? ex2_approx(fmaf(q0, -0.5f * LOG2E, r[5])) : 0.f;
                float g1 = h1 ? ex2_approx(fmaf(q1, -0.5f * LOG2E, r[5])) : 0.f;
                float G0 = -K0, G1 = -K1;
                float acc[R::V];
#pragma unroll
                for (int c = 0; c < C; c++) {
                    float m0 = r[6 + c * E], m1 = m0;
                    if (E == 3) {
                        m0 = fmaf(r[6 + c * E + 1], dx, fmaf(r[6 + c * E + 2], dy0, m0));
                        m1 = fmaf(r[6 + c * E + 1], dx, fmaf(r[6 + c * E + 2], dy1, m1));
                    }
                    G0 = fmaf(eD0[c], m0, G0);
                    G1 = fmaf(eD1[c], m1, G1);
                    float ge0 = g0 * eD0[c], ge1 = g1 * eD1[c];
                    acc[6 + c * E] = ge0 + ge1;
                    if (E == 3) {
                        acc[6 + c * E + 1] = (ge0 + ge1) * dx;
                        acc[6 + c * E + 2] = fmaf(ge0, dy0, ge1 * dy1);
                    }
                }
                float sa = g0 * G0, sb = g1 * G1;          // gG (s = -gG/2, applied in k_adam)
                float sv = fmaf(sa, w0, sb * w1);
                acc[0] = (sa + sb) * u;
                acc[1] = sv;
                acc[2] = (sa + sb) * u * dx;
                acc[3] = sv * dx;
                acc[4] = fmaf(sa * w0, dy0, sb * w1 * dy1);
                acc[5] = sa + sb;
#pragma unroll
                for (int i = R::P; i < R::V; i++) acc[i] = 0.f;
                int idx;
                float tot = warp_reduce_transpose<R::V>(acc, lane, idx);
                constexpr int GROUP = 32 / R::V;   // lanes sharing one value index
                if ((lane & (GROUP - 1)) == 0 && idx < R::P)
                    atomicAdd(&A.acc[(size_t)sid[j] * R::V + idx], tot);
            }
        }
        release();
        return;
    }

    // ---- kernel-parallel backward over per-warp pair lists ----
    // Each warp owns the (kernel, lane) entries of its 8x8 quadrant whose
    // lane has a pixel inside the kernel's ellipse, listed kernel-major in
    // shared memory (the forward wrote them while testing; larger K_n rebuild
    // them per batch).  An entry is the lane's vertical pixel pair (shared
    // dx, packed f32x2 in dy; a pixel outside the ellipse gets g = 0, so it
    // adds nothing).  The warp's 32 lanes split the list into
    // equal contiguous ranges, so every lane carries the same number of
    // entries; a lane accumulates the raw sums of the current kernel in
    // registers and flushes them with vector atomics when the kernel changes
    // and at the end of its range.
    const float4 *spw_pix = SMOE_SEED_SOA ? reinterpret_cast<const float4 *>(reinterpret_cast<const float *>(spix) + warp * 32)
                                          : spix + warp * 32 * NSEED;   // this warp's lanes' seeds
    unsigned spw_pix_s = (unsigned)__cvta_generic_to_shared(spw_pix);
    unsigned srec_s = (unsigned)__cvta_generic_to_shared(srec), sid_s = (unsigned)__cvta_generic_to_shared(sid);
    if (E == 3) {
        // linear experts: opaque copies keep the three shared bases in
        // registers instead of rematerialising them (S2UR + ULEA) at every
        // kernel switch (config 2 +1.4%; the constant-expert forms, bound to
        // 72 registers, lose 0.5-1% at configs 3/5 and stay as they are)
        asm volatile("mov.b32 %0, %0;" : "+r"(srec_s));
        asm volatile("mov.b32 %0, %0;" : "+r"(sid_s));
        asm volatile("mov.b32 %0, %0;" : "+r"(spw_pix_s));
    }
    for (int b0 = 0; b0 < n; b0 += BATCH) {
        int nb = min(BATCH, n - b0);
        int total = wrun, nr = nrec;           // n <= BATCH: listed by the forward
        if (n > BATCH) {
            load_batch(b0, nb);
            // rebuild the warp's kernel records for the resident batch
            total = 0;
            nr = 0;
            for (int j = 0; j < nb; j++) {
                float rb[R::RS];
                load_rec(j, rb);
                float dx, u;
                float2 dyv, wv, qv;
                dist2(rb, dx, dyv, u, wv, qv);
                const unsigned c0 = __ballot_sync(FULL, v0 && qv.x <= R2), c1 = __ballot_sync(FULL, v1 && qv.y <= R2);
                if ((c0 | c1) == 0u) continue;
                if (lane == 0) skr[warp][nr] = make_uint4(c0, c1, (unsigned)j, (unsigned)total);
                nr++;
                total += __popc(c0 | c1);
            }
        }
        __syncwarp();
        // lane range [lo, hi) of the warp's entries (kernel-major)
        const int lo = (lane * total) >> 5, hi = ((lane + 1) * total) >> 5;
        if (lo < hi) {
            // the record holding entry lo: last record with prefix <= lo
            int ra = 0;
            static_assert(BATCH >= 2 && BATCH <= 1024 && (BATCH & (BATCH - 1)) == 0,
                          "record search: BATCH must be a power of two");
            for (int step = BATCH / 2; step >= 1; step >>= 1)
                if (ra + step < nr && (int)skr[warp][ra + step].w <= lo) ra += step;
            uint4 kr = skr[warp][ra];
            unsigned m = kr.x | kr.y;
            {
                // drop the record's first (lo - prefix) entries: position of
                // its (k+1)-th set bit by a binary search on popcounts
                const int k = lo - (int)kr.w;
                int t = 0;
#pragma unroll
                for (int sft = 16; sft >= 1; sft >>= 1)
                    if (__popc(m & ((1u << (t + sft)) - 1u)) <= k) t += sft;
                m &= ~((1u << t) - 1u);
            }
            float4 *dst;
            float r[R::RS];
            // Raw sums of the current kernel, with gG = g G per
            // pixel (s = dL/d(d^2) = -gG/2; the -1/2 is applied in k_adam):
            //   gG u, gG v, gG u dx, gG v dx, gG v dy, gG, (g eD_c, g eD_c dx, g eD_c dy)_c
            // kept as f32x2 pairs (upper, lower pixel of the lane) and summed
            // across the pair only when flushed.
            float2 A2[R::P];
#pragma unroll
            for (int i = 0; i < R::P; i++) A2[i] = make_float2(0.f, 0.f);
            auto open_kernel = [&](int j) {
                dst = reinterpret_cast<float4 *>(A.acc + (size_t)lds32(sid_s + 4u * j) * R::V);
#pragma unroll
                for (int q4 = 0; q4 < RS4; q4++) {
                    const float4 f = lds128(srec_s + 16u * (j * RS4 + q4));
                    r[4 * q4] = f.x; r[4 * q4 + 1] = f.y; r[4 * q4 + 2] = f.z; r[4 * q4 + 3] = f.w;
                }
            };
            auto flush = [&] {
                // unpacked sums live in .x alone (.y stays +0): no x + 0 adds
                constexpr bool PEf = (SMOE_BWD_PACK & 1) != 0, PGf = (SMOE_BWD_PACK & 2) != 0;
#pragma unroll
                for (int q4 = 0; q4 < (R::P + 3) / 4; q4++) {
                    float t4[4];
#pragma unroll
                    for (int k4 = 0; k4 < 4; k4++) {
                        const int i = 4 * q4 + k4;
                        const bool packed = i < 6 ? PGf : PEf;
                        t4[k4] = i < R::P ? (packed ? A2[i].x + A2[i].y : A2[i].x) : 0.f;
                    }
                    atomicAdd(dst + q4, make_float4(t4[0], t4[1], t4[2], t4[3]));
                }
            };
            open_kernel((int)kr.z);
            for (int q = lo; q < hi; q++) {
                if (m == 0u) {
                    // kernel switch: flush this kernel's sums, open the next record
                    flush();
#pragma unroll
                    for (int i = 0; i < R::P; i++) A2[i] = make_float2(0.f, 0.f);
                    kr = skr[warp][++ra];
                    m = kr.x | kr.y;
                    open_kernel((int)kr.z);
                }
                const unsigned lb = m & (0u - m);       // lowest listed lane
                m ^= lb;
                const int l = 31 - __clz(lb);
                const bool h0 = (kr.x & lb) != 0u, h1 = (kr.y & lb) != 0u;
                // this pair's seeds and coordinates (a pixel outside the ellipse: g = 0)
                float2 ed[C], Kp, xy;
                if (SMOE_SEED_SOA) {
                    // spw_pix_s = the warp's column (warp * 32 floats); component k at + 512 k bytes
                    const unsigned a = spw_pix_s + 4u * (unsigned)l;
                    auto ld = [&](unsigned off) { return __int_as_float(lds32(a + off)); };
#pragma unroll
                    for (int c = 0; c < C; c++) ed[c] = make_float2(ld(1024u * c), ld(1024u * c + 512u));
                    Kp = make_float2(ld(1024u * C), ld(1024u * C + 512u));
                    xy = make_float2(ld(1024u * C + 1024u), ld(1024u * C + 1536u));
                } else if (C == 1) {
                    const unsigned a = spw_pix_s + (unsigned)l * (16u * NSEED);
                    const float4 p0 = lds128(a), p1 = lds128(a + 16u);
                    ed[0] = make_float2(p0.x, p0.y);
                    Kp = make_float2(p0.z, p0.w);
                    xy = make_float2(p1.x, p1.y);
                } else {
                    const unsigned a = spw_pix_s + (unsigned)l * (16u * NSEED);
                    const float4 p0 = lds128(a), p1 = lds128(a + 16u);
                    const float2 p2 = lds64(a + 32u);
                    ed[0] = make_float2(p0.x, p0.y);
                    ed[C > 1 ? 1 : 0] = make_float2(p0.z, p0.w);
                    ed[C > 2 ? 2 : 0] = make_float2(p1.x, p1.y);
                    Kp = make_float2(p1.z, p1.w);
                    xy = p2;
                }
                const float2 dd = __fadd2_rn(xy, make_float2(-r[0], -r[1]));   // (dx, dy of the upper pixel)
                const float dx = dd.x;
                const float2 dy = __fadd2_rn(make_float2(dd.y, dd.y), make_float2(0.f, 1.0f));
                const float u = r[2] * dx;
                const float bdx = r[3] * dx;
                const float2 v = __ffma2_rn(make_float2(r[4], r[4]), dy, make_float2(bdx, bdx));
                const float uu = u * u;
                const float2 qd = __ffma2_rn(v, v, make_float2(uu, uu));
                const float2 ea = __ffma2_rn(qd, make_float2(-0.5f * LOG2E, -0.5f * LOG2E), make_float2(r[5], r[5]));
                const float2 g = make_float2(h0 ? ex2_approx(ea.x) : 0.f, h1 ? ex2_approx(ea.y) : 0.f);
                // packed sums: one FFMA2/FADD2 per pair; scalar sums (in .x;
                // .y stays 0): the pair's two products added first
                constexpr bool PE = (SMOE_BWD_PACK & 1) != 0, PG = (SMOE_BWD_PACK & 2) != 0;
                float2 Gs = make_float2(-Kp.x, -Kp.y);
#pragma unroll
                for (int c = 0; c < C; c++) {
                    float2 mc = make_float2(r[6 + c * E], r[6 + c * E]);
                    if (E == 3) {
                        const float mb = fmaf(r[6 + c * E + 1], dx, r[6 + c * E]);
                        mc = __ffma2_rn(make_float2(r[6 + c * E + 2], r[6 + c * E + 2]), dy, make_float2(mb, mb));
                    }
                    Gs = __ffma2_rn(ed[c], mc, Gs);
                    float2 &am = A2[6 + c * E];
                    if (E == 3) {
                        const float2 ge = __fmul2_rn(g, ed[c]);
                        float2 &ax = A2[6 + c * E + 1], &ay = A2[6 + c * E + 2];
                        if (PE) {
                            am = __fadd2_rn(am, ge);
                            ax = __ffma2_rn(ge, make_float2(dx, dx), ax);
                            ay = __ffma2_rn(ge, dy, ay);
                        } else {
                            const float gs = ge.x + ge.y;
                            am.x += gs;
                            ax.x = fmaf(gs, dx, ax.x);
                            ay.x = fmaf(ge.x, dy.x, fmaf(ge.y, dy.y, ay.x));
                        }
                    } else if (PE) {
                        am = __ffma2_rn(g, ed[c], am);
                    } else {
                        const float2 ge = __fmul2_rn(g, ed[c]);
                        am.x += ge.x + ge.y;
                    }
                }
                const float2 gG = __fmul2_rn(g, Gs);
                const float2 sv = __fmul2_rn(gG, v);
                const float udx = u * dx;
                if (PG) {
                    A2[0] = __ffma2_rn(gG, make_float2(u, u), A2[0]);
                    A2[1] = __fadd2_rn(A2[1], sv);
                    A2[2] = __ffma2_rn(gG, make_float2(udx, udx), A2[2]);
                    A2[3] = __ffma2_rn(sv, make_float2(dx, dx), A2[3]);
                    A2[4] = __ffma2_rn(sv, dy, A2[4]);
                    A2[5] = __fadd2_rn(A2[5], gG);
                } else {
                    const float gs = gG.x + gG.y, vs = sv.x + sv.y;
                    A2[0].x = fmaf(gs, u, A2[0].x);
                    A2[1].x += vs;
                    A2[2].x = fmaf(gs, udx, A2[2].x);
                    A2[3].x = fmaf(vs, dx, A2[3].x);
                    A2[4].x = fmaf(sv.x, dy.x, fmaf(sv.y, dy.y, A2[4].x));
                    A2[5].x += gs;
                }
            }
            flush();
        }
        __syncthreads();
    }
    release();
}

// ------------------------------------------- a4, a5, a9: four pixels per lane --
// Render raster with two warps per 16x16 block: warp w covers columns
// [8w, 8w+8), lane l the vertical strip of four pixels (8w + (l & 7),
// 4 (l >> 3) + {0..3}).  The four pixels share dx, so per (warp, kernel) the
// test costs ~23 instructions for 128 pixels (two packed f32x2 pairs in dy)
// instead of ~34 for two 64-pixel warps of raster_tile (constant experts:
// ~20, with the block-centred records of SMOE_R4_XF -- the pixels then
// agree with raster_tile's render to rounding, both at the oracle bar; the
// list order, and so the summation order, is the same).
// Measured: config 3 4x SR +11%, configs 2/5 1x +6%, but config 4 1x (151
// kernels per block) -7% -- the host picks this form for grids whose
// longest bucket is short.  The same layout for the TRAIN
// raster (seeds and kernel-parallel backward over four-ballot records) was
// built, passed the parity suite and measured 8-26% slower (§10).
constexpr int R4_NT = 64;

template <int C, int E, bool PROF>
__device__ __forceinline__ void render_tile4(const RasterArgs &A, const int tile)
{
    using R = Rec<C, E>;
    constexpr int RS4 = R::RS / 4;
    constexpr int BATCH = SMOE_RASTER_BATCH;
    __shared__ float4 srec[BATCH * RS4];

    const int tx = tile % A.nx, ty = tile / A.nx;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int px = tx * TILE + warp * 8 + (lane & 7);
    const int py = ty * TILE + (lane >> 3) * 4;
    bool vv[4];
#pragma unroll
    for (int i = 0; i < 4; i++) vv[i] = px < A.oW && py + i < A.oH;
    // source coordinates of the output samples (Q16); XF (constant experts,
    // SMOE_R4_XF): relative to the block's first sample (X0, Y0), with the
    // staged records re-centred to {a, -a mx, b, -(b mx + c my), c, ...},
    // (mx, my) = mu - (X0, Y0), so the cull test is u = a x + alpha,
    // w = c y + (b x + gamma): 7 instead of 10 FP32 instructions per kernel
    constexpr bool XF = SMOE_R4_XF && E == 1;
    const float X0 = XF ? (tx * TILE + 0.5f) * A.sx - 0.5f : 0.f;
    const float Y0 = XF ? (ty * TILE + 0.5f) * A.sy - 0.5f : 0.f;
    const float xs = (px + 0.5f) * A.sx - 0.5f - X0;
    const float2 ys01 = make_float2((py + 0.5f) * A.sy - 0.5f - Y0, (py + 1.5f) * A.sy - 0.5f - Y0);
    const float2 ys23 = make_float2((py + 2.5f) * A.sy - 0.5f - Y0, (py + 3.5f) * A.sy - 0.5f - Y0);
    const float R2 = A.R2;
    const int s0 = A.len ? tile * A.bcap : A.start[tile];
    const int n = A.len ? A.len[tile] : A.start[tile + 1] - s0;
    const long long c_start = PROF ? clock64() : 0;
    constexpr int SCHUNK = (BATCH * RS4 * 4 >= 2048) ? 2048 : 1024;
    sort_bucket(A.ids + s0, n, A.tmp + s0, reinterpret_cast<int *>(srec), SCHUNK);
    if (PROF) {
        __syncthreads();
        if (threadIdx.x == 0) atomicAdd(&A.work[2], (unsigned long long)(clock64() - c_start));
    }
    float2 D01 = make_float2(0.f, 0.f), D23 = D01, N01[C], N23[C];
#pragma unroll
    for (int c = 0; c < C; c++) { N01[c] = D01; N23[c] = D01; }
    unsigned long long w_tested = 0, w_hit = 0;
    int w_valid = 0;
    if (PROF) {
#pragma unroll
        for (int i = 0; i < 4; i++) w_valid += __popc(__ballot_sync(FULL, vv[i]));
    }
    for (int b0 = 0; b0 < n; b0 += BATCH) {
        const int nb = min(BATCH, n - b0);
        __syncthreads();
        for (int i = threadIdx.x; i < nb * RS4; i += blockDim.x) {
            const int j = i / RS4, q = i - j * RS4;
            SMOE_CHECK(A.ids[s0 + b0 + j] >= 0 && A.ids[s0 + b0 + j] < A.K && (!A.len || b0 + j < A.bcap));
            srec[i] = reinterpret_cast<const float4 *>(A.rec)[(size_t)A.ids[s0 + b0 + j] * RS4 + q];
        }
        __syncthreads();
        if (XF) {
            for (int j = threadIdx.x; j < nb; j += blockDim.x) {
                const float4 f0 = srec[j * RS4];
                const float c = srec[j * RS4 + 1].x;
                const float mx = f0.x - X0, my = f0.y - Y0;
                srec[j * RS4] = make_float4(f0.z, -f0.z * mx, f0.w, -fmaf(f0.w, mx, c * my));
            }
            __syncthreads();
        }
#pragma unroll 1
        for (int j = 0; j < nb; j++) {
            float r[R::RS];
#pragma unroll
            for (int q = 0; q < RS4; q++) {
                const float4 f = srec[j * RS4 + q];
                r[4 * q] = f.x; r[4 * q + 1] = f.y; r[4 * q + 2] = f.z; r[4 * q + 3] = f.w;
            }
            float dx, u, bdx;
            float2 dy01, dy23;
            if (XF) {
                dx = 0.f; dy01 = dy23 = make_float2(0.f, 0.f);   // unused (constant experts)
                u = fmaf(r[0], xs, r[1]);
                bdx = fmaf(r[2], xs, r[3]);
                dy01 = ys01; dy23 = ys23;                          // w = c y + (b x + gamma)
            } else {
                dx = xs - r[0];
                dy01 = __fadd2_rn(ys01, make_float2(-r[1], -r[1]));
                dy23 = __fadd2_rn(ys23, make_float2(-r[1], -r[1]));
                u = r[2] * dx;
                bdx = r[3] * dx;
            }
            const float uu = u * u;
            const float2 w01 = __ffma2_rn(make_float2(r[4], r[4]), dy01, make_float2(bdx, bdx));
            const float2 w23 = __ffma2_rn(make_float2(r[4], r[4]), dy23, make_float2(bdx, bdx));
            const float2 q01 = __ffma2_rn(w01, w01, make_float2(uu, uu));
            const float2 q23 = __ffma2_rn(w23, w23, make_float2(uu, uu));
            const bool h0 = vv[0] && q01.x <= R2, h1 = vv[1] && q01.y <= R2;
            const bool h2 = vv[2] && q23.x <= R2, h3 = vv[3] && q23.y <= R2;
            if (PROF) {
                w_tested += w_valid;
                w_hit += __popc(__ballot_sync(FULL, h0)) + __popc(__ballot_sync(FULL, h1)) +
                         __popc(__ballot_sync(FULL, h2)) + __popc(__ballot_sync(FULL, h3));
            }
            if (!__any_sync(FULL, h0 || h1 || h2 || h3)) continue;
            const float2 L = make_float2(-0.5f * LOG2E, -0.5f * LOG2E), lp = make_float2(r[5], r[5]);
            const float2 e01 = __ffma2_rn(q01, L, lp), e23 = __ffma2_rn(q23, L, lp);
            const float2 g01 = make_float2(h0 ? ex2_approx(e01.x) : 0.f, h1 ? ex2_approx(e01.y) : 0.f);
            const float2 g23 = make_float2(h2 ? ex2_approx(e23.x) : 0.f, h3 ? ex2_approx(e23.y) : 0.f);
            D01 = __fadd2_rn(D01, g01);
            D23 = __fadd2_rn(D23, g23);
#pragma unroll
            for (int c = 0; c < C; c++) {
                float2 m01 = make_float2(r[6 + c * E], r[6 + c * E]), m23 = m01;
                if (E == 3) {
                    const float mb = fmaf(r[6 + c * E + 1], dx, r[6 + c * E]);
                    const float2 wy = make_float2(r[6 + c * E + 2], r[6 + c * E + 2]);
                    m01 = __ffma2_rn(wy, dy01, make_float2(mb, mb));
                    m23 = __ffma2_rn(wy, dy23, make_float2(mb, mb));
                }
                N01[c] = __ffma2_rn(g01, m01, N01[c]);
                N23[c] = __ffma2_rn(g23, m23, N23[c]);
            }
        }
    }
    if (PROF && lane == 0) {
        atomicAdd(&A.work[0], w_tested);
        atomicAdd(&A.work[1], w_hit);
    }
    // y = N/D (SMoE) or N (RBF head); each lane stores its strip (a warp
    // store covers 8 rows x 32 contiguous bytes)
    const float Dv[4] = {D01.x, D01.y, D23.x, D23.y};
    const size_t plane = (size_t)A.oH * A.oW;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        if (!vv[i]) continue;
        const float iD = A.rbf ? 1.f : (Dv[i] > 0.f ? 1.0f / Dv[i] : 0.f);
        float *o = A.out + (size_t)(py + i) * A.oW + px;
#pragma unroll
        for (int c = 0; c < C; c++) {
            const float2 Nc = (i < 2) ? N01[c] : N23[c];
            const float y = ((i & 1) ? Nc.y : Nc.x) * iD;
            o[c * plane] = A.accum != 0.f ? fmaf(A.accum, y, o[c * plane]) : y;
        }
    }
    if (A.len && threadIdx.x == 0) {
        A.lenout[tile] = n;
        if (n) A.len[tile] = 0;
    }
    if (PROF && threadIdx.x == 0) atomicAdd(&A.work[3], (unsigned long long)(clock64() - c_start));
}

template <int C, int E, bool PROF>
#ifndef SMOE_R4_MINB
#define SMOE_R4_MINB 16
#endif
__global__ void __launch_bounds__(R4_NT, SMOE_R4_MINB)
k_render4(RasterArgs A)
{
    const int tile = A.tile0 + blockIdx.x;
    if (A.gc->skip) {
        if (A.len && threadIdx.x == 0) A.len[tile] = 0;
        if (A.out) {
            const int tx = tile % A.nx, ty = tile / A.nx;
            const size_t plane = (size_t)A.oH * A.oW;
            for (int i = threadIdx.x; i < TILE * TILE; i += blockDim.x) {
                const int x = tx * TILE + (i & (TILE - 1)), y = ty * TILE + i / TILE;
                if (x < A.oW && y < A.oH)
                    for (int c = 0; c < C; c++) A.out[c * plane + (size_t)y * A.oW + x] = __int_as_float(0x7fc00000);
            }
        }
        return;
    }
    render_tile4<C, E, PROF>(A, tile);
}

// Raster grid: one CTA per block.  CTAs take the blocks in the LPT order
// written by k_preprocess (longest K_n first), boustrophedon over strata of
// n_sm consecutive CTAs (CTA b is placed on SM ~ b mod n_sm), so that every
// SM receives a mix of long and short lists when the whole grid is resident,
// and later waves start with the longest remaining lists.
template <int C, int E, bool TRAIN, bool PROF, bool KPAR>
__global__ void __launch_bounds__(128, KPAR ? (E == 3 ? SMOE_KPAR_MINB : SMOE_KPAR_MINB_CONST) : 12)
k_raster(RasterArgs A)
{
    int i = blockIdx.x;
    const int k = i / A.n_sm, j = i - k * A.n_sm;
    if ((k & 1) && (k + 1) * A.n_sm <= A.n_work) i = k * A.n_sm + (A.n_sm - 1 - j);
    const int tile = A.order ? A.order[i] : A.tile0 + i;
    if (A.gc->skip) {   // overflowed binning: no work, but the counts are reset
        if (A.len && threadIdx.x == 0) A.len[tile] = 0;
        if (!TRAIN && A.out) {
            // a skipped render leaves NaN in its output (accumulate: NaN is
            // added), never stale memory; the host reports SMOE_ERR_CAPACITY
            // at the next synchronising call and grows the lists
            const int tx = tile % A.nx, ty = tile / A.nx;
            const size_t plane = (size_t)A.oH * A.oW;
            for (int i = threadIdx.x; i < TILE * TILE; i += blockDim.x) {
                const int x = tx * TILE + (i & (TILE - 1)), y = ty * TILE + i / TILE;
                if (x < A.oW && y < A.oH)
                    for (int c = 0; c < C; c++) A.out[c * plane + (size_t)y * A.oW + x] = __int_as_float(0x7fc00000);
            }
        }
        return;
    }
    raster_tile<C, E, TRAIN, PROF, KPAR>(A, tile);
}

// ---------------------------------------------------------------- a8 ------
// MODE 0 (step):   raw sums -> parameter gradients -> Adam -> clamp; reset sums
// MODE 1 (grad):   raw sums -> parameter gradients -> grad_out; reset sums
// MODE 2 (apply):  grad_in -> Adam -> clamp
// Chain rule (DESIGN.md appendix A): the raster sums, per
// kernel, Tu = sum gG u, Tv = sum gG v, Tux = sum gG u dx, Tvx = sum gG v dx,
// Tvy = sum gG v dy, Tg = sum gG and gm_c = sum g eD_c (pixel terms with
// gG = g G = -2 s, s = dL/d(d^2)), so
//   dL/dmu_x = a Tu + b Tv - sum_c Wx_c gm_c
//   dL/dmu_y = c Tv        - sum_c Wy_c gm_c
//   dL/dl11  = a^2 Tux + a b Tvx
//   dL/dl21  = a c Tvx
//   dL/dl22  = b c Tvx + c^2 Tvy
//   dL/dlog_pi = Tg
// Adam (Q9): beta1 0.9, beta2 0.999, eps 1e-8 outside the sqrt,
// bias-corrected; clamp l11, l22 >= 1e-3.  Moments are stored
// parameter-major m[Pk][K] so every access is coalesced.
constexpr int ADAM_NT = 256;
// elements per thread of the element-parallel k_adam (used while one wave of
// resident CTAs covers every element; more per thread measured slower)
constexpr int ADAM_IT = 1;

template <int C, int E>
__device__ __forceinline__ float *param_slot(const ParamsMut &p, int k, int v)
{
    // branch-free (selects): a divergent branch per parameter group would
    // serialise the groups' load latencies
    const size_t off = v < 2 ? 2 * (size_t)k + v
                     : v < 5 ? 3 * (size_t)k + (v - 2)
                     : v == 5 ? (size_t)k : (size_t)k * C * E + (v - 6);
    float *base = v < 2 ? p.mu : v < 5 ? p.chol : v == 5 ? p.log_pi : p.expert;
    return base + off;
}

// One CTA = ADAM_IT x (ADAM_NT / V) kernels x V slots; every thread owns
// ADAM_IT (kernel, parameter) elements and issues all their loads before any
// use, so a step's loads are in flight at once.  The kernel-major raw sums and
// parameters are staged in shared memory (the chain rule of element v needs
// several of its kernel's sums and its Cholesky factor); moments and the
// update run parameter-major.
// Common arguments of the Adam kernels.  Kernels [k0, k0 + n) of the pool of
// Ktot are processed (MODE 2 on a multi-GPU kernel shard; k0 = 0, n = Ktot
// otherwise); grad_in / grad_out are [n][P] (rows relative to k0), the
// moments [P][Ktot] and the parameters absolute.
struct AdamCommon {
    int Ktot, k0, n;
    const double *skip_in;   // MODE 2: all-reduced skip flag (sums[3]); non-zero = no update
    double *dstats;          // MODE 0/1: dstats[3] = 1 when the binning overflowed
};

// An overflowed binning skipped the raster: MODE 1 writes a zero gradient
// (never stale memory) and both modes flag the skip in dstats[3], which
// smoe_grad returns as sums[3] (multi-GPU ranks all-reduce it and skip the
// update together).  Returns true when the caller must return.
template <int P, int MODE>
__device__ __forceinline__ bool adam_skipped(const AdamCommon &cm, float *grad_out, const GridCtr *gc)
{
    if (MODE == 2) return cm.skip_in && *cm.skip_in != 0.0;
    if (!gc->skip) return false;
    if (MODE == 1)
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)cm.n * P;
             i += (long long)gridDim.x * blockDim.x)
            grad_out[i] = 0.f;
    if (blockIdx.x == 0 && threadIdx.x == 0 && cm.dstats) cm.dstats[3] = 1.0;
    return true;
}

#ifndef SMOE_ADAM_MINB
#define SMOE_ADAM_MINB 6     // k_adam: min resident CTAs per SM (40 registers: config 2 Adam 11.6 -> 9.5 us,
                             // step 62.5 -> 60.9 us; config 4 neutral; 8 measured equal)
#endif
template <int C, int E, int MODE>
__global__ void __launch_bounds__(ADAM_NT, SMOE_ADAM_MINB)
k_adam(AdamCommon cm, ParamsMut p, float *__restrict__ acc, const float *__restrict__ grad_in,
       float *__restrict__ grad_out, float *__restrict__ m1, float *__restrict__ m2,
       LrDev lr, HandleCtr *hc, const GridCtr *gc, long long cap, RecOut ro)
{
    using R = Rec<C, E>;
    constexpr int P = R::P, V = R::V, KPB = ADAM_NT / V, KPC = ADAM_IT * KPB;
    __shared__ float s_raw[KPC][V + 1];
    __shared__ float s_prm[KPC][V + 1];
    if (adam_skipped<P, MODE>(cm, grad_out, gc)) return;
    const int K = cm.Ktot, k0r = cm.k0, kend = cm.k0 + cm.n;
    const long long t = hc->t + 1;
    // 1 - beta^t = -expm1(t log(beta)), accurate to a few ulp for every t
    const float bc1 = MODE == 1 ? 1.f : -expm1f((float)t * log1pf(-0.1f));
    const float bc2 = MODE == 1 ? 1.f : -expm1f((float)t * log1pf(-0.001f));
    const float rbc1 = 1.f / bc1, rbc2 = 1.f / bc2;
    bool bad = false;
    // grid-stride over chunks of KPC kernels (the host launches one CTA per
    // chunk; the loop only guards other grid sizes)
    const int nchunk = (cm.n + KPC - 1) / KPC;
    for (int chunk = blockIdx.x; chunk < nchunk; chunk += gridDim.x) {
        const int k0 = k0r + chunk * KPC;
        // every load is issued before any use: kernel-major (thread = kernel
        // kl, slot v; acc[k0*V + ...] is contiguous) for the raw sums and
        // parameters, parameter-major for the moments
        // parameter-major: thread = (parameter v, kernels kl = it*KPB + lane group)
        const int v = threadIdx.x / KPB;
        float a1[ADAM_IT], a2[ADAM_IT], gi[ADAM_IT];
#pragma unroll
        for (int it = 0; it < ADAM_IT; it++) {
            const int k = k0 + it * KPB + threadIdx.x % KPB;
            const bool live = v < P && k < kend;
            a1[it] = a2[it] = gi[it] = 0.f;
            if (live && MODE != 1) { a1[it] = m1[(size_t)v * K + k]; a2[it] = m2[(size_t)v * K + k]; }
            if (live && MODE == 2) gi[it] = grad_in[(size_t)(k - k0r) * P + v];
        }
        float rv[ADAM_IT], pv[ADAM_IT], xs[ADAM_IT];
#pragma unroll
        for (int it = 0; it < ADAM_IT; it++) {
            const int kl = it * KPB + (int)threadIdx.x / V, v = threadIdx.x % V, k = k0 + kl;
            rv[it] = pv[it] = 0.f;
            if (k < kend) {
                if (MODE != 2 && v < P) rv[it] = acc[(size_t)k0 * V + it * ADAM_NT + threadIdx.x];
                pv[it] = *param_slot<C, E>(p, k, min(v, P - 1));
            }
        }
#pragma unroll
        for (int it = 0; it < ADAM_IT; it++) {
            const int kl = it * KPB + (int)threadIdx.x / V, vv = threadIdx.x % V;
            s_raw[kl][vv] = rv[it];
            s_prm[kl][vv] = pv[it];
        }
        __syncthreads();
        if (MODE != 2) {
#pragma unroll
            for (int it = 0; it < ADAM_IT; it++)
                if (k0 + it * KPB + (int)threadIdx.x / V < kend && (int)threadIdx.x % V < P)
                    acc[(size_t)k0 * V + it * ADAM_NT + threadIdx.x] = 0.f;
        }
#pragma unroll
        for (int it = 0; it < ADAM_IT; it++) {
            const int kl = it * KPB + threadIdx.x % KPB, k = k0 + kl;
            if (!(v < P && k < kend)) continue;
            const float *raw = s_raw[kl], *prm = s_prm[kl];
            float g = gi[it];
            if (MODE != 2) {
                if (v >= 6) {
                    g = raw[v];
                } else if (v == 5) {
                    g = raw[5];
                } else {
                    const float l11 = prm[2], l21 = prm[3], l22 = prm[4];
                    const float a = 1.0f / l11, c = 1.0f / l22;
                    const float b = -l21 / (l11 * l22);
                    if (v <= 1) {
                        float ex = 0.f;
                        if (E == 3) {
#pragma unroll
                            for (int ch = 0; ch < C; ch++) ex = fmaf(prm[6 + ch * E + 1 + v], raw[6 + ch * E], ex);
                        }
                        g = (v == 0 ? fmaf(a, raw[0], b * raw[1]) : c * raw[1]) - ex;
                    } else if (v == 2) {
                        g = fmaf(a * a, raw[2], a * b * raw[3]);
                    } else if (v == 3) {
                        g = a * c * raw[3];
                    } else {
                        g = fmaf(b * c, raw[3], c * c * raw[4]);
                    }
                }
            }
            bad = bad || !isfinite(g);
            if (MODE == 1) {
                grad_out[(size_t)(k - k0r) * P + v] = g;
            } else {
                const float b1 = 0.9f, b2 = 0.999f, eps = 1e-8f;
                const float lri = v < 2 ? lr.mu : (v < 5 ? lr.chol : (v == 5 ? lr.log_pi : (((v - 6) % E) == 0 ? lr.expert : lr.slope)));
                const float n1 = fmaf(b1, a1[it], (1.f - b1) * g);
                const float n2 = fmaf(b2, a2[it], (1.f - b2) * g * g);
                float x = prm[v] - lri * (n1 * rbc1) / (sqrtf(n2 * rbc2) + eps);
                if (v == 2 || v == 4) x = fmaxf(x, 1e-3f);
                m1[(size_t)v * K + k] = n1;
                m2[(size_t)v * K + k] = n2;
                *param_slot<C, E>(p, k, v) = x;
                xs[it] = x;
            }
        }
        __syncthreads();   // shared staging is reused by the next chunk
        if (MODE != 1 && ro.rec) {
            // fused epilogue: the next step's records and tile boxes (stage 1
            // of the two-stage binning) from the parameters just written
#pragma unroll
            for (int it = 0; it < ADAM_IT; it++) {
                const int kl = it * KPB + threadIdx.x % KPB, k = k0 + kl;
                if (v < P && k < kend) s_prm[kl][v] = xs[it];
            }
            __syncthreads();
            if ((int)threadIdx.x < KPC && k0 + (int)threadIdx.x < kend) {
                const float *q = s_prm[threadIdx.x];
                write_record<C, E>(ro, k0 + threadIdx.x, make_float2(q[0], q[1]), q[2], q[3], q[4], q[5], q + 6, hc);
            }
            __syncthreads();
        }
    }
    if (bad) atomicExch((unsigned long long *)&hc->nonfinite, 1ull);
    if (MODE == 1) return;
    // the last CTA advances the step counter after every CTA has read it (the
    // reads were consumed before the barrier; no other data is published, so
    // a relaxed ticket suffices and no CTA waits for its stores to drain)
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(&hc->done, 1u) == gridDim.x - 1) {
        hc->t = t;
        hc->done = 0;
    }
}

// Large pools: one thread per kernel, all of its loads first (more bytes in
// flight per thread than the element-parallel form once several waves are
// needed; measured faster at K >= 20 000).
#ifndef SMOE_ADAMKT_MINB
#define SMOE_ADAMKT_MINB 12  // k_adam_kt: min resident 64-thread CTAs per SM (<= 80 registers, no spills;
                             // config 3 Adam 15.9 -> 13.7 us, config 5 77 -> 70 us against the uncapped
                             // 106 registers); C = 3 linear experts stay uncapped (they would spill)
#endif
template <int C, int E, int MODE>
__global__ void __launch_bounds__(64, (C == 3 && E == 3) ? 1 : SMOE_ADAMKT_MINB)
k_adam_kt(AdamCommon cm, ParamsMut p, float *__restrict__ acc, const float *__restrict__ grad_in,
       float *__restrict__ grad_out, float *__restrict__ m1, float *__restrict__ m2,
       LrDev lr, HandleCtr *hc, const GridCtr *gc, long long cap, RecOut ro)
{
    using R = Rec<C, E>;
    constexpr int P = R::P;
    if (adam_skipped<P, MODE>(cm, grad_out, gc)) return;
    const int K = cm.Ktot;
    const int kr = blockIdx.x * blockDim.x + threadIdx.x;   // row of grad_in / grad_out
    const int k = cm.k0 + kr;
    const bool live = kr < cm.n;
    const long long t = hc->t + 1;
    if (live) {
        // every load first (they are independent and overlap), then compute,
        // then every store
        float prm[P], g[P], a1[P], a2[P];
        {
            float2 mu = reinterpret_cast<const float2 *>(p.mu)[k];
            prm[0] = mu.x; prm[1] = mu.y;
            prm[2] = p.chol[3 * k]; prm[3] = p.chol[3 * k + 1]; prm[4] = p.chol[3 * k + 2];
            prm[5] = p.log_pi[k];
#pragma unroll
            for (int i = 6; i < P; i++) prm[i] = p.expert[(size_t)k * C * E + (i - 6)];
        }
        float raw[R::V];
        if (MODE == 2) {
#pragma unroll
            for (int i = 0; i < P; i++) g[i] = grad_in[(size_t)kr * P + i];
        } else {
            // only the float4 chunks holding the P sums (slots >= P are never
            // written by the raster and stay zero from the allocation)
            const float4 *ap = reinterpret_cast<const float4 *>(acc) + (size_t)k * (R::V / 4);
#pragma unroll
            for (int q = 0; q < (P + 3) / 4; q++) {
                float4 f = ap[q];
                raw[4 * q] = f.x; raw[4 * q + 1] = f.y; raw[4 * q + 2] = f.z; raw[4 * q + 3] = f.w;
            }
        }
        if (MODE != 1) {
#pragma unroll
            for (int i = 0; i < P; i++) { a1[i] = m1[(size_t)i * K + k]; a2[i] = m2[(size_t)i * K + k]; }
        }
        if (MODE != 2) {
            const float l11 = prm[2], l21 = prm[3], l22 = prm[4];
            const float a = 1.0f / l11, c = 1.0f / l22;
            const float b = -l21 / (l11 * l22);
            float ex_x = 0.f, ex_y = 0.f;
            if (E == 3) {
#pragma unroll
                for (int ch = 0; ch < C; ch++) {
                    ex_x = fmaf(prm[6 + ch * E + 1], raw[6 + ch * E], ex_x);
                    ex_y = fmaf(prm[6 + ch * E + 2], raw[6 + ch * E], ex_y);
                }
            }
            g[0] = fmaf(a, raw[0], b * raw[1]) - ex_x;
            g[1] = c * raw[1] - ex_y;
            g[2] = fmaf(a * a, raw[2], a * b * raw[3]);
            g[3] = a * c * raw[3];
            g[4] = fmaf(b * c, raw[3], c * c * raw[4]);
            g[5] = raw[5];
#pragma unroll
            for (int i = 6; i < P; i++) g[i] = raw[i];
            float4 *ap = reinterpret_cast<float4 *>(acc) + (size_t)k * (R::V / 4);
#pragma unroll
            for (int q = 0; q < (P + 3) / 4; q++) ap[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        bool ok = true;
#pragma unroll
        for (int i = 0; i < P; i++) ok = ok && isfinite(g[i]);
        if (!ok) atomicExch((unsigned long long *)&hc->nonfinite, 1ull);
        if (MODE == 1) {
#pragma unroll
            for (int i = 0; i < P; i++) grad_out[(size_t)kr * P + i] = g[i];
        } else {
            const float b1 = 0.9f, b2 = 0.999f, eps = 1e-8f;
            // 1 - beta^t = -expm1(t log(beta)), accurate to a few ulp for every t
            const float bc1 = -expm1f((float)t * log1pf(-0.1f));
            const float bc2 = -expm1f((float)t * log1pf(-0.001f));
#pragma unroll
            for (int i = 0; i < P; i++) {
                float lri = i < 2 ? lr.mu : (i < 5 ? lr.chol : (i == 5 ? lr.log_pi : (((i - 6) % E) == 0 ? lr.expert : lr.slope)));
                a1[i] = fmaf(b1, a1[i], (1.f - b1) * g[i]);
                a2[i] = fmaf(b2, a2[i], (1.f - b2) * g[i] * g[i]);
                prm[i] -= lri * (a1[i] / bc1) / (sqrtf(a2[i] / bc2) + eps);
            }
            prm[2] = fmaxf(prm[2], 1e-3f);
            prm[4] = fmaxf(prm[4], 1e-3f);
#pragma unroll
            for (int i = 0; i < P; i++) { m1[(size_t)i * K + k] = a1[i]; m2[(size_t)i * K + k] = a2[i]; }
            reinterpret_cast<float2 *>(p.mu)[k] = make_float2(prm[0], prm[1]);
            p.chol[3 * k] = prm[2]; p.chol[3 * k + 1] = prm[3]; p.chol[3 * k + 2] = prm[4];
            p.log_pi[k] = prm[5];
#pragma unroll
            for (int i = 6; i < P; i++) p.expert[(size_t)k * C * E + (i - 6)] = prm[i];
            // fused epilogue: the next step's record and tile box (stage 1 of
            // the two-stage binning) from the parameters just written
            if (ro.rec) write_record<C, E>(ro, k, make_float2(prm[0], prm[1]), prm[2], prm[3], prm[4], prm[5], prm + 6, hc);
        }
    }
    if (MODE == 1) return;
    // the last CTA advances the step counter after every CTA has read it (the
    // reads were consumed before the barrier; no other data is published, so
    // a relaxed ticket suffices and no CTA waits for its stores to drain)
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(&hc->done, 1u) == gridDim.x - 1) {
        hc->t = t;
        hc->done = 0;
    }
}

}  // namespace smoe
