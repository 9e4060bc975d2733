// smoe.cu -- host runtime and C ABI of the B200-native Rasterized SMoE path.
//
// The ABI is declared (and documented, with the paper passages it follows)
// in include/smoe.h.  This file owns the workspace, the launch sequences of
// §8(a) and the device-fault / capacity protocol.  No compute
// happens on the host: every step of the path runs in smoe_kernels.cuh.
#include "smoe.h"
#include "smoe_kernels.cuh"

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges for nsys / ncu --nvtx

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

using namespace smoe;

namespace {

struct SmoeError : std::runtime_error {
    smoe_status st;
    SmoeError(smoe_status s, const std::string &m) : std::runtime_error(m), st(s) {}
};

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            (void)cudaGetLastError();                                                     \
            throw SmoeError(e_ == cudaErrorMemoryAllocation ? SMOE_ERR_OUT_OF_MEMORY       \
                                                            : SMOE_ERR_CUDA,              \
                            std::string(#call) + ": " + cudaGetErrorString(e_));         \
        }                                                                                 \
    } while (0)

// Device-resident control block: one D2H copy brings back every counter.
struct Ctl {
    double dstats[4];   // SSE, clamped SSE, uncovered pixels, (unused)
    GridCtr train;
    GridCtr render;
    HandleCtr hc;
};

struct Prof {
    bool on = false;
    int max = 0, n = 0;
    unsigned mask = 0xffffffffu;     // kernels (bit = SMOE_KERNEL_*) to time
    std::vector<cudaEvent_t> ev;
    std::vector<int> kid;
    unsigned long long *d_work = nullptr;
};

// Arguments of one k_adam launch, kept so a captured graph's Adam node can
// be re-parameterised (new learning rates) before every replay.
struct AdamArgs {
    AdamCommon cm;
    ParamsMut pm;
    float *acc;
    const float *gin;
    float *gout;
    float *m1, *m2;
    LrDev lr;
    HandleCtr *hc;
    const GridCtr *gc;
    long long cap;
    RecOut ro;
    void *ptrs[12];
    void bind()
    {
        void *a[12] = {&cm, &pm, &acc, &gin, &gout, &m1, &m2, &lr, &hc, &gc, &cap, &ro};
        for (int i = 0; i < 12; i++) ptrs[i] = a[i];
    }
};

// A captured launch sequence (a1-a8 of smoe_step, or a1-a7 + gradient
// finalisation of smoe_grad) replayed as one CUDA graph.
struct StepGraph {
    bool valid = false;
    // key: everything baked into the captured launches
    const void *mu = nullptr, *chol = nullptr, *lp = nullptr, *ex = nullptr, *target = nullptr, *gout = nullptr;
    const int *ids = nullptr;
    long long cap = 0;
    int b0 = 0, b1 = 0, bwd = 0;
    bool prof = false;
    unsigned pmask = 0;
    bool warm = false;    // k_records omitted (records written by the previous Adam)
    bool fused = false;   // the Adam node writes the next step's records
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t adam = nullptr;
    void *adam_func = nullptr;
    dim3 adam_grid, adam_block;
    int n_kernels = 0;
    std::vector<cudaGraphNode_t> evA, evB;   // per timed launch, in launch order
    std::vector<int> evk;
};

struct Grid {
    int oH = 0, oW = 0, nx = 0, ny = 0, n_tiles = 0;
    int *cnt = nullptr, *start = nullptr, *cursor = nullptr, *order = nullptr;
    int *ids = nullptr, *tmp = nullptr;
    unsigned long long *lb_state = nullptr;   // look-back scan status words
    int *chunk = nullptr, *hist = nullptr;    // fused binning scratch
    int bin_grid = 0;                         // cooperative grid of k_bin
    bool order_valid = false;                 // LPT order written by the last binning
    // direct buckets (grids up to DIRECT_MAX blocks): block t's list is
    // ids[t bcap, t bcap + len[t]); otherwise CSR lists ids[start[t], start[t+1])
    bool direct = false;
    bool no_direct = false;   // calibration found the buckets too unbalanced for direct
    int bcap = 0;
    int *len = nullptr;
    long long cap = 0;
    bool calibrated = false;
    GridCtr *gc = nullptr;   // points into Ctl
};

}  // namespace

struct smoe_ctx {
    int K, H, W, C, order, E, P, RS, V;
    float R2;
    int device;
    cudaStream_t stream = nullptr;
    float *rec = nullptr;
    int4 *tbox = nullptr;
    float *acc = nullptr, *m1 = nullptr, *m2 = nullptr;
    Ctl *ctl = nullptr;      // device
    Ctl *h_ctl = nullptr;    // pinned host mirror
    float *stage_in = nullptr;  size_t stage_in_n = 0;
    float *stage_out = nullptr; size_t stage_out_n = 0;
    double *stage_sums = nullptr;
    Grid train, render;
    int band0 = 0, band1 = 0;   // tile rows; band1 == 0 -> whole image
    long long launches = 0;
    long long init_cap = 0;
    int bwd_mode = -1;          // -1 auto, 0 pixel-parallel, 1 kernel-parallel
    double last_pairs = -1.0;   // host view of P on the training grid (last sync)
    int n_sm = 148;
    int head = 0;               // 0 SMoE (Eq. 2/4), 1 RBF (Eq. 1)
    int box_mode = 0;           // 0 square, 1 aabb, 2 exact (reading Q4)
    // spatial kernel order of the two-stage binning (k_emit); refreshed
    // every PERM_REFRESH binnings and whenever the parameter buffer changes
    int *perm = nullptr, *perm_hist = nullptr;
    bool perm_valid = false;
    long long perm_age = 0;
    const void *perm_mu = nullptr;
    // fused records: the step's Adam wrote the next step's records and tile
    // boxes (training grid) for the parameters it updated; the next binning
    // of the same parameters and band skips k_records.  Any call that writes
    // the records, the parameters or the band clears it (invalidate_rec).
    bool rec_fresh = false;
    bool skip_records = false;
    bool fuse_now = false;      // the current sequence's Adam writes the records
    const void *rec_key[4] = {nullptr, nullptr, nullptr, nullptr};
    int rec_b0 = 0, rec_b1 = 0, rec_mode = 0;
    bool use_graphs = true;
    bool capturing = false;
    cudaStream_t cap_stream = nullptr;
    std::vector<cudaEvent_t> cap_ev;   // placeholders recorded during capture
    std::vector<int> cap_kid;
    StepGraph sg[2][4];         // graph cache per mode (step, grad), LRU by use stamp
    long long sg_use[2][4] = {{0}};
    long long sg_clock = 0;
    // host targets: double-buffered staging on a copy stream, so the H2D copy
    // of call t+1 overlaps the compute of call t
    cudaStream_t copy_stream = nullptr;
    float *tstage[2] = {nullptr, nullptr};
    cudaEvent_t tcopied[2] = {nullptr, nullptr}, tconsumed[2] = {nullptr, nullptr};
    int tslot = 0;
    int tpending = -1;          // slot whose consumption event must follow the current sequence
    Prof prof;
    std::string err;
};

namespace {

thread_local std::string g_err;

void set_err(smoe_ctx *h, const std::string &m)
{
    if (h) h->err = m;
    g_err = m;
}

// NVTX range around one ABI call (visible in nsys timelines and usable as an
// ncu --nvtx filter); a no-op unless a tool is attached.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

template <class F>
smoe_status guard(smoe_ctx *h, F &&f)
{
    try {
        if (h) CK(cudaSetDevice(h->device));
        return f();
    } catch (SmoeError &e) {
        if (h) h->rec_fresh = false;
        set_err(h, e.what());
        return e.st;
    } catch (std::bad_alloc &) {
        set_err(h, "host allocation failed");
        return SMOE_ERR_OUT_OF_MEMORY;
    } catch (std::exception &e) {
        set_err(h, e.what());
        return SMOE_ERR_CUDA;
    }
}

void check_launch(smoe_ctx *h, const char *what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw SmoeError(SMOE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    h->launches++;
}

// Launch with optional profiling events around it (same stream).
template <class F>
void launch(smoe_ctx *h, int kid, const char *what, F &&f)
{
    Prof &P = h->prof;
    bool timed = P.on && ((P.mask >> kid) & 1u);
    if (h->capturing) {
        // placeholder events; every replay swaps in fresh pool events
        int i = (int)h->cap_kid.size();
        if (timed) {
            while ((int)h->cap_ev.size() < 2 * (i + 1)) {
                cudaEvent_t e;
                CK(cudaEventCreate(&e));
                h->cap_ev.push_back(e);
            }
            CK(cudaEventRecordWithFlags(h->cap_ev[2 * i], h->stream, cudaEventRecordExternal));
        }
        f();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw SmoeError(SMOE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
        if (timed) {
            CK(cudaEventRecordWithFlags(h->cap_ev[2 * i + 1], h->stream, cudaEventRecordExternal));
            h->cap_kid.push_back(kid);
        }
        return;
    }
    bool rec = timed && P.n < P.max;
    if (rec) CK(cudaEventRecord(P.ev[2 * P.n], h->stream));
    f();
    check_launch(h, what);
    if (rec) {
        CK(cudaEventRecord(P.ev[2 * P.n + 1], h->stream));
        P.kid[P.n] = kid;
        P.n++;
    }
}

bool is_device_ptr(const void *p)
{
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

template <class T>
void dfree(T *&p)
{
    if (p) cudaFree((void *)p);
    p = nullptr;
}

void free_grid(Grid &g)
{
    dfree(g.cnt); dfree(g.start); dfree(g.cursor); dfree(g.order); dfree(g.ids); dfree(g.tmp);
    dfree(g.lb_state); dfree(g.chunk); dfree(g.hist); dfree(g.len);
    g = Grid();
}

float *stage(float *&buf, size_t &have, size_t n)
{
    if (have < n) {
        dfree(buf);
        CK(cudaMalloc(&buf, n * sizeof(float)));
        have = n;
    }
    return buf;
}

// Direct buckets up to this many blocks (measured at 129 600 and 172 890:
// config 5 preprocess 200 -> 132 us, config 3 4x render +11% over CSR lists)
constexpr long long DIRECT_MAX = 1 << 18;

void ensure_grid(smoe_ctx *h, Grid &g, GridCtr *gc, int oH, int oW)
{
    if (g.oH == oH && g.oW == oW && g.cnt) return;
    long long cap = g.cap;
    bool cal = g.calibrated && g.oH == oH && g.oW == oW;
    dfree(g.cnt); dfree(g.start); dfree(g.cursor); dfree(g.order); dfree(g.lb_state);
    dfree(g.chunk); dfree(g.hist); dfree(g.len);
    g.oH = oH; g.oW = oW;
    g.nx = (oW + TILE - 1) / TILE;
    g.ny = (oH + TILE - 1) / TILE;
    g.n_tiles = g.nx * g.ny;
    g.gc = gc;
    {
        const char *e = getenv("SMOE_CSR");
        const char *dm = getenv("SMOE_DIRECT_MAX");
        const long long direct_max = dm ? atoll(dm) : DIRECT_MAX;
        bool direct = g.n_tiles <= direct_max && !g.no_direct && !(e && atoi(e) != 0);
        if (direct != g.direct) { dfree(g.ids); dfree(g.tmp); cap = 0; cal = false; g.bcap = 0; }
        g.direct = direct;
        if (direct) {
            CK(cudaMalloc(&g.len, sizeof(int) * g.n_tiles));
            if (!cal) { dfree(g.ids); dfree(g.tmp); cap = 0; g.bcap = 0; }
        }
    }
    CK(cudaMalloc(&g.cnt, sizeof(int) * g.n_tiles));
    CK(cudaMalloc(&g.start, sizeof(int) * (g.n_tiles + 1)));
    CK(cudaMalloc(&g.cursor, sizeof(int) * g.n_tiles));
    CK(cudaMalloc(&g.order, sizeof(int) * g.n_tiles));
    CK(cudaMalloc(&g.hist, sizeof(int) * 512));

    CK(cudaMemsetAsync(g.cnt, 0, sizeof(int) * g.n_tiles, h->stream));
    CK(cudaMemsetAsync(gc, 0, sizeof(GridCtr), h->stream));
    g.cap = cap;
    g.calibrated = cal;
    g.bin_grid = 0;
    dfree(g.chunk);
}

void grow(smoe_ctx *h, Grid &g, long long need)
{
    h->rec_fresh = false;   // the redo bins from scratch
    long long cap = need + need / 4 + 4096;
    if (g.direct) {
        // need = the longest bucket; every block gets the same capacity
        long long b = (need + need / 4 + 32 + 31) / 32 * 32;
        if (b * g.n_tiles >= (1ll << 31)) throw SmoeError(SMOE_ERR_OUT_OF_MEMORY, "bucket capacity beyond 2^31 ids");
        g.bcap = (int)b;
        cap = b * g.n_tiles;
    }
    dfree(g.ids); dfree(g.tmp);
    CK(cudaMalloc(&g.ids, sizeof(int) * cap));
    CK(cudaMalloc(&g.tmp, sizeof(int) * cap));
    // defined contents for the slots past a bucket's length (read only by the
    // smoe_bin diagnostic copy; keeps compute-sanitizer initcheck clean)
    CK(cudaMemsetAsync(g.ids, 0, sizeof(int) * cap, h->stream));
    CK(cudaMemsetAsync(g.tmp, 0, sizeof(int) * cap, h->stream));
    g.cap = cap;
    g.calibrated = true;
    CK(cudaMemsetAsync(&g.gc->need, 0, 2 * sizeof(long long), h->stream));  // need, skipped
    CK(cudaMemsetAsync(&g.gc->skip, 0, sizeof(unsigned), h->stream));       // the calibrating binning's latch
}

void read_ctl(smoe_ctx *h)
{
    CK(cudaMemcpyAsync(h->h_ctl, h->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (h->h_ctl->train.pairs > 0) h->last_pairs = (double)h->h_ctl->train.pairs;
}

// Backward form: the kernel-parallel pass over per-warp
// pixel-pair lists, unless the caller forces the pixel-parallel pass with
// warp reductions (smoe_options.backward_mode = 0).
int effective_bwd(smoe_ctx *h)
{
    // auto: kernel-parallel (measured faster at 23-604 kernels per block,
    // configs 1-5 and a config-4 density sweep; scripts/gpu_density.sh)
    return h->bwd_mode >= 0 ? h->bwd_mode : 1;
}

#define DISPATCH_CE(h, BODY)                                                  \
    do {                                                                      \
        if (h->C == 1 && h->E == 1) { constexpr int C_ = 1, E_ = 1; BODY; }   \
        else if (h->C == 1 && h->E == 3) { constexpr int C_ = 1, E_ = 3; BODY; } \
        else if (h->C == 3 && h->E == 1) { constexpr int C_ = 3, E_ = 1; BODY; } \
        else { constexpr int C_ = 3, E_ = 3; BODY; }                          \
    } while (0)

// LPT block order: built by the preprocess's last CTA for grids up to
// SCAN_SINGLE_MAX blocks (larger grids run several waves where the hardware
// scheduler balances, and use the look-back scan).
#ifndef SMOE_LPT
#define SMOE_LPT 1
#endif
bool use_lpt(const Grid &g) { return SMOE_LPT && !g.lb_state && g.n_tiles <= SCAN_SINGLE_MAX && !getenv("SMOE_NO_LPT"); }

ParamsDev pdev(const smoe_params *p) { return ParamsDev{p->mu, p->chol, p->log_pi, p->expert}; }

BoxGeo box_geo(const smoe_ctx *h, const Grid &g)
{
    return BoxGeo{h->box_mode, (float)h->W / (float)g.oW, (float)h->H / (float)g.oH, g.oW, g.oH};
}

void check_params(const smoe_params *p)
{
    if (!p || !p->mu || !p->chol || !p->log_pi || !p->expert)
        throw SmoeError(SMOE_ERR_INVALID_ARG, "params: NULL pointer");
    if (!is_device_ptr(p->mu) || !is_device_ptr(p->chol) || !is_device_ptr(p->log_pi) || !is_device_ptr(p->expert))
        throw SmoeError(SMOE_ERR_INVALID_ARG, "params must be device pointers");
    if (((uintptr_t)p->mu & 7) != 0) throw SmoeError(SMOE_ERR_INVALID_ARG, "params.mu must be 8-byte aligned");
}

// a1-a4: preprocess, scan, scatter, in-bucket sort on grid g for block rows
// [ty_lo, ty_hi).  The first binning of a grid calibrates the capacity with
// one synchronous read of P; later binnings never synchronise.
// Two-stage binning (k_records + k_emit over a spatial kernel order) for
// large pools on direct-bucket grids: one returning global atomic per
// (CTA, block) instead of per (kernel, block).  SMOE_PERM=0/1 forces it off/on.
constexpr int RENDER4_MAX_BCAP = 256;   // render form switch (bucket capacity = 1.25 x longest + 32)
constexpr int PRE_TPK = 8;   // one-pass direct binning: threads per kernel (measured: config 2 +4%, config 1 +3% over 1)
constexpr int PERM_MIN_K = 16384;   // measured: config 4 (20k) +6%, config 2 (10k) -2%
constexpr long long PERM_REFRESH = 256;

bool two_stage(const smoe_ctx *h, const Grid &g)
{
    const char *e = getenv("SMOE_PERM");
    const bool on = e ? atoi(e) != 0 : h->K >= PERM_MIN_K;
    return on && g.direct;
}

// (Re)build the spatial order: counting sort of the kernel centres into
// square buckets of ~256 kernels.  Eager launches on the
// handle's stream, before any graph replay that reads the order.
void refresh_perm(smoe_ctx *h, const smoe_params *p, bool force)
{
    const char *e = getenv("SMOE_PERM");
    const bool on = e ? atoi(e) != 0 : h->K >= PERM_MIN_K;
    if (!on) return;
    if (!force && h->perm_valid && h->perm_mu == p->mu && h->perm_age < PERM_REFRESH) return;
    if (!h->perm) {
        CK(cudaMalloc(&h->perm, sizeof(int) * h->K));
        CK(cudaMalloc(&h->perm_hist, sizeof(int) * PERM_MAX_BUCKETS));
    }
    const double tiles = std::ceil(h->W / 16.0) * std::ceil(h->H / 16.0);
    int side = 16 * std::max(1, (int)std::lround(std::sqrt(tiles / std::max(1.0, h->K / 256.0))));
    int nbx, nby;
    for (;; side *= 2) {
        nbx = (h->W + side - 1) / side;
        nby = (h->H + side - 1) / side;
        if ((long long)nbx * nby <= PERM_MAX_BUCKETS) break;
    }
    const float scale = 1.0f / (float)side;
    const int nb = (h->K + 255) / 256;
    CK(cudaMemsetAsync(h->perm_hist, 0, sizeof(int) * nbx * nby, h->stream));
    k_perm_count<<<nb, 256, 0, h->stream>>>(h->K, p->mu, scale, scale, nbx, nby, h->perm_hist);
    check_launch(h, "k_perm_count");
    k_perm_scan<<<1, PERM_NT, 0, h->stream>>>(h->perm_hist, nbx * nby);
    check_launch(h, "k_perm_scan");
    k_perm_scatter<<<nb, 256, 0, h->stream>>>(h->K, p->mu, scale, scale, nbx, nby, h->perm_hist, h->perm);
    check_launch(h, "k_perm_scatter");
    h->perm_valid = true;
    h->perm_age = 0;
    h->perm_mu = p->mu;
}

void bin_unfused(smoe_ctx *h, Grid &g, const smoe_params *p, int ty_lo, int ty_hi, bool zero_stats, float lscale)
{
    int K = h->K;
    if (two_stage(h, g) && h->perm_valid) {
        float sx = (float)g.oW / (float)h->W, sy = (float)g.oH / (float)h->H;
        const int nb = (K + PRE_NT - 1) / PRE_NT;
        if (!(&g == &h->train && h->skip_records))
            launch(h, SMOE_KERNEL_PREPROCESS, "k_records", [&] {
                DISPATCH_CE(h, (k_records<C_, E_><<<nb, PRE_NT, 0, h->stream>>>(
                                   K, pdev(p), h->R2, sx, sy, g.oW, g.oH, g.nx, ty_lo, ty_hi, h->rec, h->tbox,
                                   &h->ctl->hc, lscale, h->box_mode)));
            });
        const int ne = (K + EMIT_NT - 1) / EMIT_NT;
        launch(h, SMOE_KERNEL_EMIT, "k_emit", [&] {
            k_emit<<<ne, EMIT_NT, 0, h->stream>>>(K, h->perm, h->tbox, g.nx, ty_lo, ty_hi, g.cnt, g.ids, g.bcap,
                                                   g.gc, zero_stats ? h->ctl->dstats : nullptr, h->rec, h->RS / 4,
                                                   box_geo(h, g), h->R2);
        });
        if (!g.calibrated) {
            long long cn[2];   // pairs, need
            CK(cudaMemcpyAsync(cn, &g.gc->pairs, sizeof(cn), cudaMemcpyDeviceToHost, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            if (&g == &h->train) h->last_pairs = (double)cn[0];
            CK(cudaMemsetAsync(g.cnt, 0, sizeof(int) * g.n_tiles, h->stream));
            if (g.n_tiles > SCAN_SINGLE_MAX && cn[1] * (long long)g.n_tiles > 8 * cn[0] + (1ll << 24)) {
                g.no_direct = true;
                const int oH = g.oH, oW = g.oW;
                g.oH = 0;
                ensure_grid(h, g, g.gc, oH, oW);
                return bin_unfused(h, g, p, ty_lo, ty_hi, zero_stats, lscale);
            }
            grow(h, g, cn[1] > 0 ? cn[1] : 1);
            return bin_unfused(h, g, p, ty_lo, ty_hi, zero_stats, lscale);
        }
        g.order_valid = false;
        return;
    }
    // direct buckets need no CTA-wide block pass, so smaller CTAs spread the
    // count atomics over more SMs
    static const int pre_nt_direct = getenv("SMOE_PRE_NT_DIRECT") ? atoi(getenv("SMOE_PRE_NT_DIRECT")) : PRE_NT;
    const int pre_nt = g.direct ? pre_nt_direct : PRE_NT;
    // direct buckets: threads per kernel (SMOE_PRE_TPK overrides)
    const char *te = getenv("SMOE_PRE_TPK");
    const int tpk = g.direct ? std::max(1, te ? atoi(te) : PRE_TPK) : 1;
    int nb = (int)(((long long)K * tpk + pre_nt - 1) / pre_nt);
    float sx = (float)g.oW / (float)h->W, sy = (float)g.oH / (float)h->H;
    if (!g.direct && g.n_tiles > SCAN_SINGLE_MAX && !g.lb_state) {
        size_t nbl = (g.n_tiles + LB_CHUNK - 1) / LB_CHUNK;
        CK(cudaMalloc(&g.lb_state, sizeof(unsigned long long) * nbl));
        CK(cudaMemsetAsync(g.lb_state, 0, sizeof(unsigned long long) * nbl, h->stream));
    }
    launch(h, SMOE_KERNEL_PREPROCESS, "k_preprocess", [&] {
        DISPATCH_CE(h, (k_preprocess<C_, E_><<<nb, pre_nt, 0, h->stream>>>(
                           K, pdev(p), h->R2, sx, sy, g.oW, g.oH, g.nx, ty_lo, ty_hi, h->rec, h->tbox,
                           g.cnt, &h->ctl->hc, g.n_tiles, g.start, g.cursor, g.cap, g.gc,
                           zero_stats ? h->ctl->dstats : nullptr, g.lb_state ? nullptr : g.order, lscale,
                           use_lpt(g) ? 1 : 0, g.ids, g.bcap, g.direct ? g.len : nullptr, h->box_mode, tpk)));
    });
    if (g.direct) {
        if (!g.calibrated) {
            // every slot overflowed (capacity 0): size the buckets from the
            // longest one, then bin again (the counts were reset)
            long long cn[2];   // pairs, need
            CK(cudaMemcpyAsync(cn, &g.gc->pairs, sizeof(cn), cudaMemcpyDeviceToHost, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            if (&g == &h->train) h->last_pairs = (double)cn[0];
            // no raster consumed this binning: reset its counts
            CK(cudaMemsetAsync(g.cnt, 0, sizeof(int) * g.n_tiles, h->stream));
            if (g.n_tiles > SCAN_SINGLE_MAX && cn[1] * (long long)g.n_tiles > 8 * cn[0] + (1ll << 24)) {
                // fixed-capacity buckets would be mostly empty: CSR lists instead
                g.no_direct = true;
                const int oH = g.oH, oW = g.oW;
                g.oH = 0;
                ensure_grid(h, g, g.gc, oH, oW);
                return bin_unfused(h, g, p, ty_lo, ty_hi, zero_stats, lscale);
            }
            grow(h, g, cn[1] > 0 ? cn[1] : 1);
            return bin_unfused(h, g, p, ty_lo, ty_hi, zero_stats, lscale);
        }
        g.order_valid = false;   // direct buckets: identity block order
        return;
    }
    if (g.lb_state) {
        int nb2 = (g.n_tiles + LB_CHUNK - 1) / LB_CHUNK;
        launch(h, SMOE_KERNEL_SCAN, "k_scan_lookback", [&] {
            k_scan_lookback<<<nb2, LB_NT, 0, h->stream>>>(g.cnt, g.n_tiles, g.start, g.cursor, g.cap, g.gc,
                                                           zero_stats ? h->ctl->dstats : nullptr, g.lb_state);
        });
    }
    if (!g.calibrated) {
        long long P;
        CK(cudaMemcpyAsync(&P, &g.gc->pairs, sizeof(P), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        if (&g == &h->train) h->last_pairs = (double)P;
        grow(h, g, P > h->init_cap ? P : h->init_cap);
    }
    int ns = (K + 63) / 64;
    launch(h, SMOE_KERNEL_SCATTER, "k_scatter", [&] {
        k_scatter<<<ns, 64, 0, h->stream>>>(K, h->tbox, g.nx, ty_lo, ty_hi, g.cursor, g.ids, g.cap, g.gc, h->rec,
                                             h->RS / 4, box_geo(h, g), h->R2);
    });
    g.order_valid = use_lpt(g);
}

// a1-a4 binning of grid g for block rows [ty_lo, ty_hi): one cooperative
// k_bin launch, or k_preprocess (+ k_scan_lookback) + k_scatter.  The
// cooperative launch costs a few us more than a plain one (measured), so the
// fused form is used for large pools (K >= 50000: config 3 gains 3%);
// SMOE_FUSED_BIN=0/1 forces either.  The first binning of a grid calibrates
// the capacity with one synchronous read of P; later binnings never sync.
void bin(smoe_ctx *h, Grid &g, const smoe_params *p, int ty_lo, int ty_hi, bool zero_stats, float lscale = 1.0f)
{
    const char *fe = getenv("SMOE_FUSED_BIN");
    bool fused = !g.direct && (fe ? atoi(fe) != 0 : h->K >= 50000);
    if (!fused) return bin_unfused(h, g, p, ty_lo, ty_hi, zero_stats, lscale);
    int K = h->K;
    if (!g.bin_grid) {
        int occ = 0;
        const void *f = nullptr;
        DISPATCH_CE(h, (f = (const void *)k_bin<C_, E_>));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, BIN_NT, 0));
        int want = std::max((K + BIN_NT - 1) / BIN_NT, (g.n_tiles + BIN_NT - 1) / BIN_NT);
        g.bin_grid = std::max(1, std::min(want, std::max(1, occ) * h->n_sm));
        CK(cudaMalloc(&g.chunk, sizeof(int) * g.bin_grid));
    }
    BinArgs B{};
    B.K = K; B.p = pdev(p); B.R2 = h->R2;
    B.sx = (float)g.oW / (float)h->W; B.sy = (float)g.oH / (float)h->H; B.lscale = lscale;
    B.oW = g.oW; B.oH = g.oH; B.nx = g.nx; B.ty_lo = ty_lo; B.ty_hi = ty_hi; B.n_tiles = g.n_tiles;
    B.rec = h->rec; B.tbox = h->tbox; B.cnt = g.cnt; B.start = g.start; B.cursor = g.cursor; B.ids = g.ids;
    B.order = SMOE_LPT && !getenv("SMOE_NO_LPT") ? g.order : nullptr;
    B.chunk = g.chunk; B.hist = g.hist; B.cap = g.cap; B.gc = g.gc; B.hc = &h->ctl->hc;
    B.dstats = zero_stats ? h->ctl->dstats : nullptr;
    B.mode = h->box_mode;
    B.rs4 = h->RS / 4;
    launch(h, SMOE_KERNEL_BIN, "k_bin", [&] {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(g.bin_grid);
        cfg.blockDim = dim3(BIN_NT);
        cfg.stream = h->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        DISPATCH_CE(h, ((void)cudaLaunchKernelEx(&cfg, k_bin<C_, E_>, B)));
    });
    g.order_valid = B.order != nullptr;
    if (!g.calibrated) {
        // the scatter phase skipped (capacity 0): size the lists, then scatter
        long long P;
        CK(cudaMemcpyAsync(&P, &g.gc->pairs, sizeof(P), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        if (&g == &h->train) h->last_pairs = (double)P;
        grow(h, g, P > h->init_cap ? P : h->init_cap);
        int ns = (K + 63) / 64;
        launch(h, SMOE_KERNEL_SCATTER, "k_scatter", [&] {
            k_scatter<<<ns, 64, 0, h->stream>>>(K, h->tbox, g.nx, ty_lo, ty_hi, g.cursor, g.ids, g.cap, g.gc,
                                                 h->rec, h->RS / 4, box_geo(h, g), h->R2);
        });
        g.order_valid = false;
    }
}

void band_rows(smoe_ctx *h, int &ty_lo, int &ty_hi)
{
    int ny = (h->H + TILE - 1) / TILE;
    if (h->band1 > h->band0) { ty_lo = h->band0; ty_hi = h->band1; }
    else { ty_lo = 0; ty_hi = ny; }
}

const float *stage_target(smoe_ctx *h, const float *target)
{
    if (is_device_ptr(target)) return target;
    size_t n = (size_t)h->C * h->H * h->W;
    if (!h->copy_stream) {
        CK(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
        for (int i = 0; i < 2; i++) {
            CK(cudaMalloc(&h->tstage[i], n * sizeof(float)));
            CK(cudaEventCreateWithFlags(&h->tcopied[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&h->tconsumed[i], cudaEventDisableTiming));
            CK(cudaEventRecord(h->tconsumed[i], h->stream));
        }
    }
    const int s = h->tslot;
    h->tslot ^= 1;
    CK(cudaStreamWaitEvent(h->copy_stream, h->tconsumed[s], 0));      // buffer no longer read
    int ty_lo, ty_hi;
    band_rows(h, ty_lo, ty_hi);
    const int r0 = ty_lo * TILE, r1 = std::min(ty_hi * TILE, h->H);
    if (r0 == 0 && r1 == h->H) {
        CK(cudaMemcpyAsync(h->tstage[s], target, n * sizeof(float), cudaMemcpyHostToDevice, h->copy_stream));
    } else {
        // a band reads only its own pixel rows: copy those, one row of the
        // 2D copy per channel (pitch H*W floats)
        const size_t off = (size_t)r0 * h->W, pitch = (size_t)h->H * h->W * sizeof(float);
        CK(cudaMemcpy2DAsync(h->tstage[s] + off, pitch, target + off, pitch,
                             (size_t)(r1 - r0) * h->W * sizeof(float), h->C, cudaMemcpyHostToDevice,
                             h->copy_stream));
    }
    CK(cudaEventRecord(h->tcopied[s], h->copy_stream));
    CK(cudaStreamWaitEvent(h->stream, h->tcopied[s], 0));
    h->tpending = s;
    return h->tstage[s];
}

// After the launch sequence that read a staged target: mark its buffer free.
void release_target(smoe_ctx *h)
{
    if (h->tpending >= 0) {
        CK(cudaEventRecord(h->tconsumed[h->tpending], h->stream));
        h->tpending = -1;
    }
}

// a1-a7 on the training grid (current band): raw sums into h->acc, loss
// partials into ctl->dstats.
void forward_backward(smoe_ctx *h, const smoe_params *p, const float *target)
{
    Grid &g = h->train;
    ensure_grid(h, g, &h->ctl->train, h->H, h->W);
    int ty_lo, ty_hi;
    band_rows(h, ty_lo, ty_hi);
    bin(h, g, p, ty_lo, ty_hi, true);
    int nt = (ty_hi - ty_lo) * g.nx;
    if (nt <= 0) return;
    RasterArgs A{};
    A.K = h->K;
    A.rec = h->rec; A.ids = g.ids; A.tmp = g.tmp; A.start = g.start; A.gc = g.gc; A.cap = g.cap;
    A.len = g.direct ? g.cnt : nullptr; A.lenout = g.len; A.bcap = g.bcap;
    A.order = g.order_valid ? g.order : nullptr;
    A.gcw = g.gc; A.n_work = nt; A.n_sm = h->n_sm;
    A.nx = g.nx; A.tile0 = ty_lo * g.nx; A.oW = h->W; A.oH = h->H;
    A.sx = 1.0f; A.sy = 1.0f; A.R2 = h->R2; A.rbf = h->head;
    A.target = target;
    A.e_scale = (float)(2.0 / ((double)h->H * h->W * h->C));
    A.acc = h->acc; A.dstats = h->ctl->dstats; A.out = nullptr;
    A.work = h->prof.d_work;
    launch(h, SMOE_KERNEL_RASTER_TRAIN, "k_raster<train>", [&] {
        bool kp = effective_bwd(h) == 1;
        bool cw = h->prof.on && (h->prof.mask & 0x80000000u);
        const void *f = nullptr;
        if (cw && kp) DISPATCH_CE(h, (f = (const void *)k_raster<C_, E_, true, true, true>));
        else if (kp) DISPATCH_CE(h, (f = (const void *)k_raster<C_, E_, true, false, true>));
        else if (cw) DISPATCH_CE(h, (f = (const void *)k_raster<C_, E_, true, true, false>));
        else DISPATCH_CE(h, (f = (const void *)k_raster<C_, E_, true, false, false>));
        void *args[1] = {&A};
        (void)cudaLaunchKernel(f, dim3(nt), dim3(128), args, 0, h->stream);
    });
}

// k_adam (element-parallel) while one wave of resident CTAs (8 per SM)
// covers every (kernel, slot) element, else k_adam_kt (one thread per kernel)
static bool adam_elementwise(smoe_ctx *h)
{
    int v = 0;
    DISPATCH_CE(h, (v = Rec<C_, E_>::V));
    return (long long)h->K <= 8LL * h->n_sm * (ADAM_NT / v);
}

void *adam_func(smoe_ctx *h, int mode)
{
    void *f = nullptr;
    if (adam_elementwise(h)) {
        if (mode == 0) DISPATCH_CE(h, (f = (void *)k_adam<C_, E_, 0>));
        else if (mode == 1) DISPATCH_CE(h, (f = (void *)k_adam<C_, E_, 1>));
        else DISPATCH_CE(h, (f = (void *)k_adam<C_, E_, 2>));
    } else {
        if (mode == 0) DISPATCH_CE(h, (f = (void *)k_adam_kt<C_, E_, 0>));
        else if (mode == 1) DISPATCH_CE(h, (f = (void *)k_adam_kt<C_, E_, 1>));
        else DISPATCH_CE(h, (f = (void *)k_adam_kt<C_, E_, 2>));
    }
    return f;
}

// Fused records: on when the training grid uses the two-stage
// binning (SMOE_FUSE_REC=0 turns it off).
bool fuse_rec(smoe_ctx *h)
{
    const char *e = getenv("SMOE_FUSE_REC");
    const bool on = !e || atoi(e) != 0;
    return on && h->train.calibrated && h->train.oH == h->H && h->train.oW == h->W && two_stage(h, h->train) &&
           h->perm_valid;
}

RecOut rec_out(smoe_ctx *h)
{
    int ty_lo, ty_hi;
    band_rows(h, ty_lo, ty_hi);
    return RecOut{h->rec, h->tbox, h->R2, h->W, h->H, ty_lo, ty_hi, h->box_mode, h->K};
}

bool rec_is_fresh(const smoe_ctx *h, const smoe_params *p)
{
    return h->rec_fresh && h->rec_key[0] == p->mu && h->rec_key[1] == p->chol && h->rec_key[2] == p->log_pi &&
           h->rec_key[3] == p->expert && h->rec_b0 == h->band0 && h->rec_b1 == h->band1 &&
           h->rec_mode == h->box_mode;
}

void mark_rec_fresh(smoe_ctx *h, const smoe_params *p)
{
    h->rec_fresh = true;
    h->rec_key[0] = p->mu; h->rec_key[1] = p->chol; h->rec_key[2] = p->log_pi; h->rec_key[3] = p->expert;
    h->rec_b0 = h->band0; h->rec_b1 = h->band1; h->rec_mode = h->box_mode;
}

void invalidate_rec(smoe_ctx *h) { h->rec_fresh = false; }

void adam_args(smoe_ctx *h, const smoe_params *p, const float *grad_in, float *grad_out, const smoe_lr *lr,
               AdamArgs &a, int k0 = 0, int n = -1, const double *skip_in = nullptr, bool fused = false)
{
    a.cm.Ktot = h->K;
    a.cm.k0 = k0;
    a.cm.n = n < 0 ? h->K : n;
    a.cm.skip_in = skip_in;
    a.cm.dstats = h->ctl->dstats;
    a.pm = ParamsMut{p->mu, p->chol, p->log_pi, p->expert};
    a.acc = h->acc;
    a.gin = grad_in;
    a.gout = grad_out;
    a.m1 = h->m1;
    a.m2 = h->m2;
    a.lr = lr ? LrDev{lr->mu, lr->chol, lr->log_pi, lr->expert, lr->slope} : LrDev{0, 0, 0, 0, 0};
    a.hc = &h->ctl->hc;
    a.gc = &h->ctl->train;
    a.cap = h->train.cap;
    a.ro = fused ? rec_out(h) : RecOut{nullptr, nullptr, 0.f, 0, 0, 0, 0, 0};
    a.bind();
}

void launch_adam(smoe_ctx *h, int mode, const smoe_params *p, const float *grad_in, float *grad_out,
                 const smoe_lr *lr, int k0 = 0, int n = -1, const double *skip_in = nullptr, bool fused = false)
{
    AdamArgs a;
    adam_args(h, p, grad_in, grad_out, lr, a, k0, n, skip_in, fused);
    void *f = adam_func(h, mode);
    dim3 grid, block;
    const int cnt = std::max(1, a.cm.n);
    if (adam_elementwise(h)) {
        int kpb = 0;
        DISPATCH_CE(h, (kpb = ADAM_NT / Rec<C_, E_>::V));
        grid = dim3((cnt + kpb - 1) / kpb);
        block = dim3(ADAM_NT);
    } else {
        grid = dim3((cnt + 63) / 64);
        block = dim3(64);
    }
    launch(h, SMOE_KERNEL_ADAM, "k_adam", [&] {
        (void)cudaLaunchKernel(f, grid, block, a.ptrs, 0, h->stream);
    });
}

// Inspect the latched device faults after a synchronisation point.
smoe_status faults(smoe_ctx *h, Grid *g_overflow_report = nullptr)
{
    Ctl &c = *h->h_ctl;
    if (c.hc.nonfinite) {
        CK(cudaMemsetAsync(&h->ctl->hc.nonfinite, 0, sizeof(long long), h->stream));
        set_err(h, "non-finite parameter or gradient detected on the device");
        return SMOE_ERR_NONFINITE;
    }
    smoe_status st = SMOE_OK;
    Grid *gs[2] = {&h->train, &h->render};
    GridCtr *cs[2] = {&c.train, &c.render};
    for (int i = 0; i < 2; i++) {
        if (cs[i]->need > (gs[i]->direct ? gs[i]->bcap : gs[i]->cap) && gs[i]->ids) {
            long long skipped = cs[i]->skipped;
            grow(h, *gs[i], cs[i]->need);
            set_err(h, "pair capacity exceeded; grown to " + std::to_string(gs[i]->cap) + ", " +
                           std::to_string(skipped) + " call(s) skipped");
            st = SMOE_ERR_CAPACITY;
        }
    }
    (void)g_overflow_report;
    return st;
}

void fill_stats(smoe_ctx *h, smoe_stats *s)
{
    Ctl &c = *h->h_ctl;
    double n = (double)h->H * h->W * h->C;
    s->sse = c.dstats[0];
    s->sse_clamped = c.dstats[1];
    s->uncovered_px = (long long)c.dstats[2];
    s->loss = c.dstats[0] / n;
    double mse_c = c.dstats[1] / n;
    s->psnr_db = mse_c > 0 ? 10.0 * std::log10(1.0 / mse_c) : INFINITY;
    s->pairs = c.train.pairs;
    s->n_tiles = h->train.n_tiles;
}

void destroy_graph(StepGraph &g)
{
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
    g = StepGraph();
}

bool graph_matches(smoe_ctx *h, const StepGraph &g, const smoe_params *p, const float *t, float *gout)
{
    return g.valid && g.mu == p->mu && g.chol == p->chol && g.lp == p->log_pi && g.ex == p->expert &&
           g.target == t && g.gout == gout && g.ids == h->train.ids && g.cap == h->train.cap &&
           g.b0 == h->band0 && g.b1 == h->band1 &&
           g.bwd == effective_bwd(h) && g.prof == h->prof.on && g.pmask == h->prof.mask &&
           g.warm == h->skip_records && g.fused == h->fuse_now;
}

// Capture forward_backward + k_adam(mode) on the private capture stream.
void capture(smoe_ctx *h, StepGraph &g, int mode, const smoe_params *p, const float *t, float *gout,
             const smoe_lr *lr)
{
    destroy_graph(g);
    if (!h->cap_stream) CK(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
    cudaStream_t user = h->stream;
    h->stream = h->cap_stream;
    h->capturing = true;
    h->cap_kid.clear();
    long long launches0 = h->launches;
    cudaGraph_t graph = nullptr;
    CK(cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
    try {
        forward_backward(h, p, t);
        launch_adam(h, mode, p, nullptr, gout, lr, 0, -1, nullptr, h->fuse_now);
    } catch (...) {
        cudaStreamEndCapture(h->cap_stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        h->stream = user;
        h->capturing = false;
        throw;
    }
    cudaError_t e = cudaStreamEndCapture(h->cap_stream, &graph);
    h->stream = user;
    h->capturing = false;
    h->launches = launches0;
    if (e != cudaSuccess) throw SmoeError(SMOE_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    g.graph = graph;
    CK(cudaGraphInstantiate(&g.exec, graph, 0));
    size_t nn = 0;
    CK(cudaGraphGetNodes(graph, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    CK(cudaGraphGetNodes(graph, nodes.data(), &nn));
    size_t nt = h->cap_kid.size();
    g.evA.assign(nt, nullptr);
    g.evB.assign(nt, nullptr);
    g.evk = h->cap_kid;
    g.adam_func = adam_func(h, mode);
    g.n_kernels = 0;
    for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType ty;
        CK(cudaGraphNodeGetType(nd, &ty));
        if (ty == cudaGraphNodeTypeKernel) {
            cudaKernelNodeParams kp;
            CK(cudaGraphKernelNodeGetParams(nd, &kp));
            g.n_kernels++;
            if (kp.func == g.adam_func) { g.adam = nd; g.adam_grid = kp.gridDim; g.adam_block = kp.blockDim; }
        } else if (ty == cudaGraphNodeTypeEventRecord) {
            cudaEvent_t ev;
            CK(cudaGraphEventRecordNodeGetEvent(nd, &ev));
            for (size_t i = 0; i < nt; i++) {
                if (h->cap_ev[2 * i] == ev) g.evA[i] = nd;
                if (h->cap_ev[2 * i + 1] == ev) g.evB[i] = nd;
            }
        }
    }
    if (!g.adam) throw SmoeError(SMOE_ERR_CUDA, "graph capture: Adam node not found");
    g.mu = p->mu; g.chol = p->chol; g.lp = p->log_pi; g.ex = p->expert;
    g.target = t; g.gout = gout; g.ids = h->train.ids; g.cap = h->train.cap;
    g.b0 = h->band0; g.b1 = h->band1; g.bwd = effective_bwd(h);
    g.prof = h->prof.on; g.pmask = h->prof.mask;
    g.warm = h->skip_records; g.fused = h->fuse_now;
    g.valid = true;
}

// Replay: new learning rates into the Adam node, fresh profiling events, launch.
void replay(smoe_ctx *h, StepGraph &g, const smoe_params *p, float *gout, const smoe_lr *lr)
{
    AdamArgs a;
    adam_args(h, p, nullptr, gout, lr, a, 0, -1, nullptr, g.fused);
    cudaKernelNodeParams kp = {};
    kp.func = g.adam_func;
    kp.gridDim = g.adam_grid;
    kp.blockDim = g.adam_block;
    kp.sharedMemBytes = 0;
    kp.kernelParams = a.ptrs;
    kp.extra = nullptr;
    CK(cudaGraphExecKernelNodeSetParams(g.exec, g.adam, &kp));
    Prof &P = h->prof;
    if (g.prof) {
        for (size_t i = 0; i < g.evk.size(); i++) {
            if (P.n >= P.max || !g.evA[i] || !g.evB[i]) break;
            CK(cudaGraphExecEventRecordNodeSetEvent(g.exec, g.evA[i], P.ev[2 * P.n]));
            CK(cudaGraphExecEventRecordNodeSetEvent(g.exec, g.evB[i], P.ev[2 * P.n + 1]));
            P.kid[P.n] = g.evk[i];
            P.n++;
        }
    }
    CK(cudaGraphLaunch(g.exec, h->stream));
    h->launches += g.n_kernels;
}

// One step (mode 0) or gradient pass (mode 1): graph replay once the grid
// is calibrated, eager launches otherwise.
struct SeqFlags {
    smoe_ctx *h;
    ~SeqFlags() { h->skip_records = h->fuse_now = false; }
};

void run_sequence(smoe_ctx *h, int mode, const smoe_params *p, const float *t, float *gout, const smoe_lr *lr)
{
    // fused records: skip k_records when the previous step's Adam wrote them
    // for these parameters; this step's Adam (mode 0) writes the next ones
    const bool fuse = fuse_rec(h);
    SeqFlags flags_{h};
    h->skip_records = fuse && rec_is_fresh(h, p);
    h->fuse_now = fuse && mode == 0;
    invalidate_rec(h);
    bool ready = h->use_graphs && h->train.calibrated && h->train.oH == h->H && h->train.oW == h->W &&
                 h->train.cnt != nullptr;
    if (!ready) {
        forward_backward(h, p, t);
        launch_adam(h, mode, p, nullptr, gout, lr, 0, -1, nullptr, h->fuse_now);
        release_target(h);
        // mode 1 leaves the parameters (and the records just used) as they were
        if (fuse) mark_rec_fresh(h, p);
        return;
    }
    // graph cache lookup (key: buffers, band, modes); evict the least recent
    int hit = -1, lru = 0;
    for (int i = 0; i < 4; i++) {
        if (graph_matches(h, h->sg[mode][i], p, t, gout)) hit = i;
        if (h->sg_use[mode][i] < h->sg_use[mode][lru]) lru = i;
    }
    if (hit < 0) {
        hit = lru;
        capture(h, h->sg[mode][hit], mode, p, t, gout, lr);
    }
    h->sg_use[mode][hit] = ++h->sg_clock;
    replay(h, h->sg[mode][hit], p, gout, lr);
    release_target(h);
    if (fuse) mark_rec_fresh(h, p);
}

}  // namespace

// ============================================================== C ABI =====
extern "C" {

int smoe_abi_version(void) { return SMOE_ABI_VERSION; }

const char *smoe_status_string(smoe_status s)
{
    switch (s) {
    case SMOE_OK: return "ok";
    case SMOE_ERR_INVALID_ARG: return "invalid argument";
    case SMOE_ERR_CUDA: return "CUDA error";
    case SMOE_ERR_OUT_OF_MEMORY: return "out of memory";
    case SMOE_ERR_NONFINITE: return "non-finite value";
    case SMOE_ERR_CAPACITY: return "pair capacity exceeded";
    case SMOE_ERR_BAD_HANDLE: return "bad handle";
    }
    return "unknown status";
}

const char *smoe_last_error(smoe_handle h) { return h ? h->err.c_str() : g_err.c_str(); }

smoe_status smoe_default_options(smoe_options *o)
{
    if (!o) return SMOE_ERR_INVALID_ARG;
    std::memset(o, 0, sizeof(*o));
    o->C = 3;
    o->R2 = 2.0 * std::log(100.0);   // chi2_2(0.99) (Q1)
    o->device = -1;
    o->use_graphs = 1;
    o->backward_mode = -1;
    o->box_mode = 1;   // aabb: measured faster than the square box on fitted pools
    return SMOE_OK;
}

smoe_lr smoe_paper_lr(int t, int T)
{
    smoe_lr l;
    double frac = T > 0 ? (double)t / T : 0.0;
    l.mu = (float)(0.01 * std::pow(1e-3, frac));   // 0.01 -> 1e-5
    l.chol = 1e-3f;
    l.log_pi = 0.0f;                               // Q11 frozen
    l.expert = 1e-3f;
    l.slope = 2e-4f;                               // Q13
    return l;
}

smoe_status smoe_create_ex(const smoe_options *o, smoe_handle *out)
{
    if (!o || !out) { g_err = "NULL argument"; return SMOE_ERR_INVALID_ARG; }
    *out = nullptr;
    if (o->K < 1 || o->H < 1 || o->W < 1 || !(o->C == 1 || o->C == 3) ||
        !(o->expert_order == 0 || o->expert_order == 1) || !(o->R2 > 0) ||
        !(o->backward_mode >= -1 && o->backward_mode <= 1) || !(o->head == 0 || o->head == 1) ||
        !(o->box_mode >= 0 && o->box_mode <= 2)) {
        g_err = "smoe_create: need K,H,W >= 1, C in {1,3}, expert_order in {0,1}, R2 > 0, box_mode in {0,1,2}";
        return SMOE_ERR_INVALID_ARG;
    }
    if ((long long)o->H * o->W >= (1ll << 31) || o->K >= (1 << 30)) {
        g_err = "smoe_create: image or kernel count too large";
        return SMOE_ERR_INVALID_ARG;
    }
    smoe_ctx *h = new (std::nothrow) smoe_ctx();
    if (!h) return SMOE_ERR_OUT_OF_MEMORY;
    h->K = o->K; h->H = o->H; h->W = o->W; h->C = o->C; h->order = o->expert_order;
    h->E = 1 + 2 * h->order;
    h->P = 6 + h->C * h->E;
    h->RS = (h->P + 3) & ~3;
    h->V = h->P <= 8 ? 8 : 16;
    h->R2 = (float)o->R2;
    h->init_cap = o->pair_capacity;
    h->bwd_mode = o->backward_mode;
    h->head = o->head;
    h->box_mode = o->box_mode;
    h->use_graphs = o->use_graphs != 0;
    int dev = o->device;
    if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) {
        (void)cudaGetLastError();
        g_err = "no CUDA device";
        delete h;
        return SMOE_ERR_CUDA;
    }
    h->device = dev;
    smoe_status st = guard(h, [&]() {
        size_t K = h->K;
        CK(cudaDeviceGetAttribute(&h->n_sm, cudaDevAttrMultiProcessorCount, h->device));
        CK(cudaMalloc(&h->rec, K * h->RS * sizeof(float)));
        CK(cudaMalloc(&h->tbox, K * sizeof(int4)));
        CK(cudaMalloc(&h->acc, K * h->V * sizeof(float)));
        CK(cudaMalloc(&h->m1, K * h->P * sizeof(float)));
        CK(cudaMalloc(&h->m2, K * h->P * sizeof(float)));
        CK(cudaMalloc(&h->ctl, sizeof(Ctl)));
        CK(cudaMallocHost(&h->h_ctl, sizeof(Ctl)));
        CK(cudaMalloc(&h->stage_sums, 4 * sizeof(double)));
        CK(cudaMemset(h->acc, 0, K * h->V * sizeof(float)));
        CK(cudaMemset(h->m1, 0, K * h->P * sizeof(float)));
        CK(cudaMemset(h->m2, 0, K * h->P * sizeof(float)));
        CK(cudaMemset(h->ctl, 0, sizeof(Ctl)));
        std::memset(h->h_ctl, 0, sizeof(Ctl));
        CK(cudaDeviceSynchronize());
        return SMOE_OK;
    });
    if (st != SMOE_OK) {
        g_err = h->err;
        smoe_destroy(h);
        return st;
    }
    *out = h;
    return SMOE_OK;
}

smoe_status smoe_create(int K, int H, int W, int C, int expert_order, smoe_handle *out)
{
    smoe_options o;
    smoe_default_options(&o);
    o.K = K; o.H = H; o.W = W; o.C = C; o.expert_order = expert_order;
    return smoe_create_ex(&o, out);
}

smoe_status smoe_destroy(smoe_handle h)
{
    if (!h) return SMOE_ERR_BAD_HANDLE;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    else cudaDeviceSynchronize();
    free_grid(h->train);
    free_grid(h->render);
    dfree(h->rec); dfree(h->tbox); dfree(h->acc); dfree(h->m1); dfree(h->m2);
    dfree(h->ctl); dfree(h->stage_in); dfree(h->stage_out); dfree(h->stage_sums);
    if (h->h_ctl) cudaFreeHost(h->h_ctl);
    for (cudaEvent_t e : h->prof.ev) cudaEventDestroy(e);
    for (cudaEvent_t e : h->cap_ev) cudaEventDestroy(e);
    for (int m = 0; m < 2; m++)
        for (int i = 0; i < 4; i++) destroy_graph(h->sg[m][i]);
    if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
    for (int i = 0; i < 2; i++) {
        dfree(h->tstage[i]);
        if (h->tcopied[i]) cudaEventDestroy(h->tcopied[i]);
        if (h->tconsumed[i]) cudaEventDestroy(h->tconsumed[i]);
    }
    if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
    dfree(h->prof.d_work);
    dfree(h->perm);
    dfree(h->perm_hist);
    (void)cudaGetLastError();
    delete h;
    return SMOE_OK;
}

smoe_status smoe_set_stream(smoe_handle h, void *stream)
{
    if (!h) return SMOE_ERR_BAD_HANDLE;
    h->stream = (cudaStream_t)stream;
    return SMOE_OK;
}

smoe_status smoe_set_band(smoe_handle h, int r0, int r1)
{
    if (!h) return SMOE_ERR_BAD_HANDLE;
    int ny = (h->H + TILE - 1) / TILE;
    if (r0 == 0 && r1 == 0) { h->band0 = h->band1 = 0; return SMOE_OK; }
    if (r0 < 0 || r1 > ny || r0 >= r1) {
        set_err(h, "smoe_set_band: need 0 <= row0 < row1 <= ceil(H/16)");
        return SMOE_ERR_INVALID_ARG;
    }
    h->band0 = r0; h->band1 = r1;
    return SMOE_OK;
}

smoe_status smoe_invalidate(smoe_handle h)
{
    if (!h) return SMOE_ERR_BAD_HANDLE;
    h->rec_fresh = false;
    return SMOE_OK;
}

smoe_status smoe_reset_adam(smoe_handle h)
{
    if (!h) return SMOE_ERR_BAD_HANDLE;
    return guard(h, [&]() {
        CK(cudaMemsetAsync(h->m1, 0, (size_t)h->K * h->P * sizeof(float), h->stream));
        CK(cudaMemsetAsync(h->m2, 0, (size_t)h->K * h->P * sizeof(float), h->stream));
        CK(cudaMemsetAsync(&h->ctl->hc, 0, sizeof(HandleCtr), h->stream));
        return SMOE_OK;
    });
}

smoe_status smoe_sync(smoe_handle h, smoe_stats *last)
{
    if (!h) return SMOE_ERR_BAD_HANDLE;
    return guard(h, [&]() {
        read_ctl(h);
        if (last) fill_stats(h, last);
        return faults(h);
    });
}

smoe_status smoe_step(smoe_handle h, smoe_params *p, const float *target, const smoe_lr *lr,
                      smoe_stats *stats)
{
    NvtxRange nvtx_("smoe_step");
    if (!h) return SMOE_ERR_BAD_HANDLE;
    return guard(h, [&]() -> smoe_status {
        check_params(p);
        if (!target || !lr) throw SmoeError(SMOE_ERR_INVALID_ARG, "smoe_step: NULL target or lr");
        refresh_perm(h, p, false);
        h->perm_age++;
        for (int attempt = 0;; attempt++) {
            const float *t = stage_target(h, target);
            run_sequence(h, 0, p, t, nullptr, lr);
            if (!stats) return SMOE_OK;
            read_ctl(h);
            smoe_status st = faults(h);
            if (st == SMOE_ERR_CAPACITY && attempt < 3) continue;   // grown: redo the skipped step
            fill_stats(h, stats);
            return st;
        }
    });
}

smoe_status smoe_grad(smoe_handle h, const smoe_params *p, const float *target, float *grad, double *sums)
{
    NvtxRange nvtx_("smoe_grad");
    if (!h) return SMOE_ERR_BAD_HANDLE;
    return guard(h, [&]() -> smoe_status {
        check_params(p);
        if (!target || !grad) throw SmoeError(SMOE_ERR_INVALID_ARG, "smoe_grad: NULL target or grad");
        refresh_perm(h, p, false);
        h->perm_age++;
        bool gdev = is_device_ptr(grad);
        bool sdev = sums ? is_device_ptr(sums) : true;
        for (int attempt = 0;; attempt++) {
            const float *t = stage_target(h, target);
            size_t n = (size_t)h->K * h->P;
            float *gout = gdev ? grad : stage(h->stage_out, h->stage_out_n, n);
            run_sequence(h, 1, p, t, gout, nullptr);
            if (gdev && sdev) {
                if (sums)
                    CK(cudaMemcpyAsync(sums, h->ctl->dstats, 4 * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
                return SMOE_OK;
            }
            read_ctl(h);
            smoe_status st = faults(h);
            if (st == SMOE_ERR_CAPACITY && attempt < 3) continue;
            if (!gdev) {
                CK(cudaMemcpyAsync(grad, gout, n * sizeof(float), cudaMemcpyDeviceToHost, h->stream));
                CK(cudaStreamSynchronize(h->stream));
            }
            if (sums) {
                if (sdev) CK(cudaMemcpy(sums, h->ctl->dstats, 4 * sizeof(double), cudaMemcpyDeviceToDevice));
                else std::memcpy(sums, h->h_ctl->dstats, 4 * sizeof(double));
            }
            return st;
        }
    });
}

smoe_status smoe_apply(smoe_handle h, smoe_params *p, const float *grad, const smoe_lr *lr)
{
    if (!h) return SMOE_ERR_BAD_HANDLE;
    return smoe_apply_ex(h, p, grad, lr, 0, h->K, nullptr);
}

smoe_status smoe_apply_ex(smoe_handle h, smoe_params *p, const float *grad, const smoe_lr *lr, int k0, int k1,
                          const double *sums)
{
    NvtxRange nvtx_("smoe_apply");
    if (!h) return SMOE_ERR_BAD_HANDLE;
    return guard(h, [&]() -> smoe_status {
        check_params(p);
        if (!grad || !lr) throw SmoeError(SMOE_ERR_INVALID_ARG, "smoe_apply: NULL grad or lr");
        if (k0 < 0 || k1 > h->K || k0 > k1) throw SmoeError(SMOE_ERR_INVALID_ARG, "smoe_apply_ex: need 0 <= k0 <= k1 <= K");
        const double *skip = nullptr;
        if (sums) {
            if (is_device_ptr(sums)) {
                skip = sums + 3;
            } else if (sums[3] != 0.0) {
                return SMOE_OK;   // a rank skipped its band: no update anywhere
            }
        }
        if (k1 == k0) return SMOE_OK;
        invalidate_rec(h);   // parameters change outside a step
        const float *g = grad;
        size_t n = (size_t)(k1 - k0) * h->P;
        if (!is_device_ptr(grad)) {
            float *d = stage(h->stage_in, h->stage_in_n, n);
            CK(cudaMemcpyAsync(d, grad, n * sizeof(float), cudaMemcpyHostToDevice, h->stream));
            g = d;
        }
        launch_adam(h, 2, p, g, nullptr, lr, k0, k1 - k0, skip);
        return SMOE_OK;
    });
}

smoe_status smoe_render(smoe_handle h, const smoe_params *p, int out_H, int out_W, float *out)
{
    return smoe_render_ex(h, p, out_H, out_W, out, nullptr);
}

smoe_status smoe_render_ex(smoe_handle h, const smoe_params *p, int out_H, int out_W, float *out,
                           const smoe_render_options *opt)
{
    NvtxRange nvtx_("smoe_render");
    if (!h) return SMOE_ERR_BAD_HANDLE;
    return guard(h, [&]() -> smoe_status {
        check_params(p);
        if (!out || out_H < 1 || out_W < 1 || (long long)out_H * out_W >= (1ll << 31))
            throw SmoeError(SMOE_ERR_INVALID_ARG, "smoe_render: bad output");
        float sharpen = opt ? opt->sharpen : 1.0f;
        if (!(sharpen > 0.0f && sharpen <= 1.0f))
            throw SmoeError(SMOE_ERR_INVALID_ARG, "smoe_render: sharpen must be in (0, 1]");
        float lscale = sqrtf(sharpen);
        invalidate_rec(h);   // the render binning overwrites the records and tile boxes
        refresh_perm(h, p, false);
        h->perm_age++;
        bool odev = is_device_ptr(out);
        if (!odev && opt && opt->accumulate != 0.0f)
            throw SmoeError(SMOE_ERR_INVALID_ARG, "smoe_render_ex: accumulate needs a device output");
        for (int attempt = 0;; attempt++) {
            Grid &g = h->render;
            ensure_grid(h, g, &h->ctl->render, out_H, out_W);
            bin(h, g, p, 0, g.ny, false, lscale);
            size_t n = (size_t)h->C * out_H * out_W;
            float *o = odev ? out : stage(h->stage_out, h->stage_out_n, n);
            RasterArgs A{};
            A.K = h->K;
            A.rec = h->rec; A.ids = g.ids; A.tmp = g.tmp; A.start = g.start; A.gc = g.gc; A.cap = g.cap;
            A.len = g.direct ? g.cnt : nullptr; A.lenout = g.len; A.bcap = g.bcap;
            A.order = g.order_valid ? g.order : nullptr; A.gcw = g.gc; A.n_work = g.n_tiles; A.n_sm = h->n_sm;
            A.nx = g.nx; A.tile0 = 0; A.oW = out_W; A.oH = out_H;
            A.sx = (float)h->W / (float)out_W; A.sy = (float)h->H / (float)out_H;
            A.R2 = h->R2; A.out = o; A.rbf = h->head;
            A.accum = opt ? opt->accumulate : 0.0f;
            A.vec_out = opt && opt->vector_stores ? 1 : 0;
            A.work = h->prof.d_work;
            // four pixels per lane for grids whose longest bucket is short
            // (measured: +6 to +11% at <= ~110 kernels per block, -7% at config
            // 4's 151); SMOE_RENDER4=0/1 forces either form
            const char *r4e = getenv("SMOE_RENDER4");
            const bool r4 = !A.order && !A.vec_out && (r4e ? atoi(r4e) != 0 : (g.direct && g.bcap <= RENDER4_MAX_BCAP));
            launch(h, SMOE_KERNEL_RASTER_RENDER, "k_raster<render>", [&] {
                const void *f = nullptr;
                if (r4) {
                    if (h->prof.on && (h->prof.mask & 0x80000000u))
                        DISPATCH_CE(h, (f = (const void *)k_render4<C_, E_, true>));
                    else DISPATCH_CE(h, (f = (const void *)k_render4<C_, E_, false>));
                    void *args[1] = {&A};
                    (void)cudaLaunchKernel(f, dim3(g.n_tiles), dim3(R4_NT), args, 0, h->stream);
                    return;
                }
                if (h->prof.on && (h->prof.mask & 0x80000000u))
                    DISPATCH_CE(h, (f = (const void *)k_raster<C_, E_, false, true, false>));
                else DISPATCH_CE(h, (f = (const void *)k_raster<C_, E_, false, false, false>));
                void *args[1] = {&A};
                (void)cudaLaunchKernel(f, dim3(g.n_tiles), dim3(128), args, 0, h->stream);
            });
            if (odev) return SMOE_OK;
            read_ctl(h);
            smoe_status st = faults(h);
            if (st == SMOE_ERR_CAPACITY && attempt < 3) continue;
            CK(cudaMemcpyAsync(out, o, n * sizeof(float), cudaMemcpyDeviceToHost, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            return st;
        }
    });
}

smoe_status smoe_bin(smoe_handle h, const smoe_params *p, int out_H, int out_W, int *tile_range, int *ids,
                     long long ids_cap, long long *n_pairs, int *tilebox)
{
    if (!h) return SMOE_ERR_BAD_HANDLE;
    if (out_H < 1 || out_W < 1) { set_err(h, "smoe_bin: bad raster"); return SMOE_ERR_INVALID_ARG; }
    // The lists are reported exactly as the hot path leaves them: a render
    // on the out_H x out_W raster bins (a1-a3) and its raster CTAs sort their
    // buckets in place (a4).
    smoe_status st = guard(h, [&]() -> smoe_status {
        size_t n = (size_t)h->C * out_H * out_W;
        float *scratch = nullptr;
        CK(cudaMalloc(&scratch, n * sizeof(float)));
        smoe_status s2 = smoe_render(h, p, out_H, out_W, scratch);
        if (s2 == SMOE_OK) {
            read_ctl(h);
            s2 = faults(h);
        }
        cudaFree(scratch);
        return s2;
    });
    if (st != SMOE_OK) return st;
    return guard(h, [&]() -> smoe_status {
        Grid &g = h->render;
        long long P = h->h_ctl->render.pairs;
        if (n_pairs) *n_pairs = P;
        if (ids && ids_cap < P) throw SmoeError(SMOE_ERR_INVALID_ARG, "smoe_bin: ids_cap < P");
        if (g.direct) {
            // direct buckets -> the CSR form of the ABI
            std::vector<int> len(g.n_tiles), all((size_t)g.n_tiles * g.bcap), st(g.n_tiles + 1), cs;
            CK(cudaMemcpy(len.data(), g.len, sizeof(int) * g.n_tiles, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(all.data(), g.ids, sizeof(int) * all.size(), cudaMemcpyDeviceToHost));
            cs.reserve((size_t)P);
            for (int t = 0; t < g.n_tiles; t++) {
                st[t] = (int)cs.size();
                cs.insert(cs.end(), all.begin() + (size_t)t * g.bcap, all.begin() + (size_t)t * g.bcap + len[t]);
            }
            st[g.n_tiles] = (int)cs.size();
            if (tile_range) CK(cudaMemcpy(tile_range, st.data(), sizeof(int) * st.size(), cudaMemcpyDefault));
            if (ids && !cs.empty()) CK(cudaMemcpy(ids, cs.data(), sizeof(int) * cs.size(), cudaMemcpyDefault));
        } else {
            if (tile_range) CK(cudaMemcpy(tile_range, g.start, sizeof(int) * (g.n_tiles + 1), cudaMemcpyDefault));
            if (ids) CK(cudaMemcpy(ids, g.ids, sizeof(int) * P, cudaMemcpyDefault));
        }
        if (tilebox) CK(cudaMemcpy(tilebox, h->tbox, sizeof(int4) * h->K, cudaMemcpyDefault));
        return SMOE_OK;
    });
}

long long smoe_launch_count(smoe_handle h) { return h ? h->launches : -1; }

smoe_status smoe_get_adam(smoe_handle h, float *m1, float *m2, long long *t)
{
    if (!h) return SMOE_ERR_BAD_HANDLE;
    if (!m1 || !m2 || !t) { set_err(h, "smoe_get_adam: NULL argument"); return SMOE_ERR_INVALID_ARG; }
    return guard(h, [&]() {
        size_t n = (size_t)h->K * h->P;
        CK(cudaStreamSynchronize(h->stream));
        // library layout is parameter-major [Pk][K]; the ABI layout is [K][Pk]
        std::vector<float> a(n), b(n);
        CK(cudaMemcpy(a.data(), h->m1, n * sizeof(float), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(b.data(), h->m2, n * sizeof(float), cudaMemcpyDeviceToHost));
        std::vector<float> ta(n), tb(n);
        for (int i = 0; i < h->P; i++)
            for (int k = 0; k < h->K; k++) {
                ta[(size_t)k * h->P + i] = a[(size_t)i * h->K + k];
                tb[(size_t)k * h->P + i] = b[(size_t)i * h->K + k];
            }
        CK(cudaMemcpy(m1, ta.data(), n * sizeof(float), cudaMemcpyDefault));
        CK(cudaMemcpy(m2, tb.data(), n * sizeof(float), cudaMemcpyDefault));
        HandleCtr hc;
        CK(cudaMemcpy(&hc, &h->ctl->hc, sizeof(hc), cudaMemcpyDeviceToHost));
        *t = hc.t;
        return SMOE_OK;
    });
}

smoe_status smoe_set_adam(smoe_handle h, const float *m1, const float *m2, long long t)
{
    if (!h) return SMOE_ERR_BAD_HANDLE;
    if (!m1 || !m2 || t < 0) { set_err(h, "smoe_set_adam: bad argument"); return SMOE_ERR_INVALID_ARG; }
    return guard(h, [&]() {
        size_t n = (size_t)h->K * h->P;
        std::vector<float> a(n), b(n), ta(n), tb(n);
        CK(cudaMemcpy(a.data(), m1, n * sizeof(float), cudaMemcpyDefault));
        CK(cudaMemcpy(b.data(), m2, n * sizeof(float), cudaMemcpyDefault));
        for (int i = 0; i < h->P; i++)
            for (int k = 0; k < h->K; k++) {
                ta[(size_t)i * h->K + k] = a[(size_t)k * h->P + i];
                tb[(size_t)i * h->K + k] = b[(size_t)k * h->P + i];
            }
        CK(cudaStreamSynchronize(h->stream));
        CK(cudaMemcpy(h->m1, ta.data(), n * sizeof(float), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(h->m2, tb.data(), n * sizeof(float), cudaMemcpyHostToDevice));
        HandleCtr hc{};
        hc.t = t;
        CK(cudaMemcpy(&h->ctl->hc, &hc, sizeof(hc), cudaMemcpyHostToDevice));
        return SMOE_OK;
    });
}

smoe_status smoe_stats_async(smoe_handle h, smoe_raw_stats *dst)
{
    if (!h) return SMOE_ERR_BAD_HANDLE;
    if (!dst) { set_err(h, "smoe_stats_async: NULL dst"); return SMOE_ERR_INVALID_ARG; }
    return guard(h, [&]() {
        CK(cudaMemcpyAsync(&dst->sse, h->ctl->dstats, 3 * sizeof(double), cudaMemcpyDefault, h->stream));
        CK(cudaMemcpyAsync(&dst->pairs, &h->ctl->train.pairs, sizeof(long long), cudaMemcpyDefault, h->stream));
        return SMOE_OK;
    });
}

smoe_status smoe_stats_from_raw(smoe_handle h, const smoe_raw_stats *raw, smoe_stats *out)
{
    if (!h) return SMOE_ERR_BAD_HANDLE;
    if (!raw || !out) return SMOE_ERR_INVALID_ARG;
    double n = (double)h->H * h->W * h->C;
    out->sse = raw->sse;
    out->sse_clamped = raw->sse_clamped;
    out->uncovered_px = (long long)raw->uncovered;
    out->loss = raw->sse / n;
    double mse_c = raw->sse_clamped / n;
    out->psnr_db = mse_c > 0 ? 10.0 * std::log10(1.0 / mse_c) : INFINITY;
    out->pairs = raw->pairs;
    out->n_tiles = h->train.n_tiles;
    return SMOE_OK;
}

const char *smoe_kernel_name(int id)
{
    static const char *names[SMOE_KERNEL_COUNT] = {"k_preprocess", "k_scatter", "k_raster<train>",
                                                   "k_raster<render>", "k_adam", "k_bin", "k_scan_lookback",
                                                   "k_emit"};
    return (id >= 0 && id < SMOE_KERNEL_COUNT) ? names[id] : "?";
}

smoe_status smoe_profile_begin(smoe_handle h, int max_launches, unsigned kernel_mask)
{
    if (!h) return SMOE_ERR_BAD_HANDLE;
    if (max_launches < 1) { set_err(h, "max_launches < 1"); return SMOE_ERR_INVALID_ARG; }
    return guard(h, [&]() {
        Prof &P = h->prof;
        while ((int)P.ev.size() < 2 * max_launches) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            P.ev.push_back(e);
        }
        P.kid.assign(max_launches, -1);
        P.max = max_launches;
        P.n = 0;
        P.mask = kernel_mask ? kernel_mask : 0xffffffffu;
        if (!P.d_work) CK(cudaMalloc(&P.d_work, 4 * sizeof(unsigned long long)));
        CK(cudaMemsetAsync(P.d_work, 0, 4 * sizeof(unsigned long long), h->stream));
        P.on = true;
        return SMOE_OK;
    });
}

smoe_status smoe_profile_end(smoe_handle h, smoe_kernel_time *times, smoe_work *work)
{
    if (!h) return SMOE_ERR_BAD_HANDLE;
    return guard(h, [&]() {
        Prof &P = h->prof;
        CK(cudaStreamSynchronize(h->stream));
        if (times) {
            for (int i = 0; i < SMOE_KERNEL_COUNT; i++) times[i] = smoe_kernel_time{0.0, 0};
            for (int i = 0; i < P.n; i++) {
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, P.ev[2 * i], P.ev[2 * i + 1]));
                times[P.kid[i]].total_ms += ms;
                times[P.kid[i]].launches += 1;
            }
        }
        if (work) {
            unsigned long long w[4] = {0, 0, 0, 0};
            if (P.d_work) CK(cudaMemcpy(w, P.d_work, sizeof(w), cudaMemcpyDeviceToHost));
            work->tested_pairs = (long long)w[0];
            work->hit_pairs = (long long)w[1];
            work->sort_cycles = (long long)w[2];
            work->cta_cycles = (long long)w[3];
        }
        P.on = false;
        P.n = 0;
        return SMOE_OK;
    });
}

}  // extern "C"
