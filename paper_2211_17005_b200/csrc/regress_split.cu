// regress_split.cu -- K5 with the layer-0 split: the SGD step
// and the full-sample evaluation of the backward regression (regressor.cpp:
// 97-158, 191-213) for the paper's network (two hidden layers of U = 64),
// without a feature matrix.
//
// A feature row of replica (k, l) at step i (labels.cpp:142-167) is
// [1{s_klc <= i} for the Cc clients, y_k] where y_k -- rates, FX, client
// intensities, lagged rates, standardised -- is the same for all N replicas
// of path k.  So layer 0 splits:
//     z0 = (b0 + W0_y y_k) + W0_ind 1{s_kl <= i}
// P_k = b0 + W0_y y_k is computed once per path of a tile (FP32 FMA chains
// over the q columns), the indicator part from the replica's default steps
// (uint16 per name).  Per 128-row tile the kernel reads 8 default steps and a
// label per row plus one y_k per path -- ~3 KB instead of a 24 KB feature
// tile -- and the step never materialises the 2M x 48 feature matrix.
//
// k_sgd_split<ACT>  the whole SGD gradient in one launch, one CTA per SM
//   (persistent over the batch's tiles, 512 TMEM columns, ~226 KB of shared
//   memory).  Per tile (thread r = row r = TMEM lane r, two warpgroups of 32
//   columns):
//     H1 = act(P_k + W0_ind ind)     SIMT; act'(H1) kept in registers;
//                                    H1 hi|lo -> TMEM (A), H1^T hi|lo -> smem
//     F1   D  = H1 W1^T              (M=128, N=64, K=64, A in TMEM)
//          H2, f, residual, G2 = dd w2 act'(H2); G2 hi|lo -> TMEM, G2^T -> smem
//     B    D  = G2 W1                (B: the W1^T tile)
//     gW1 += G2^T [H1^T; 1]          (M=64, N=72, K=128 rows, both SW128 smem)
//          G1 = D act'(H1); G1^T hi|lo -> smem
//     Dind = G1^T [ind; member]      (M=64, N=32, K=128: indicator columns and
//                                     per-path row sums, exact 0/1 operand)
//          gW0_ind += Dind[:, c];  s_p = Dind[:, 8+p];  gb0 += s_p;
//          gW0_y += s_p (x) y_p      (SIMT, 64 owner threads)
//   so the weight gradients accumulate in tensor memory / registers across
//   the CTA's tiles and leave once, as one FP32 partial row per CTA (no
//   transposed activations in HBM, no second kernel).  3xTF32 throughout.
// k_eval_split<ACT>  loss / head-switch minimum / predictions / layer-2
//   activations, two CTAs per SM: P for every path of the tile (N >= 1),
//   H1 -> TMEM, F1, epilogue as k_eval_tc.
// Reductions are over fixed tile -> CTA maps in fixed order: deterministic.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "regress_act.cuh"
#include "regress_opt.cuh"
#include "regress_tc.cuh"
#include "tc.cuh"

namespace hcva {
namespace {

constexpr int kU = 64;           // hidden width served here
constexpr int kQ = 48;           // per-path columns (q <= 48), row stride of ysh
constexpr int kInd = 8;          // indicator columns (Cc <= 8)
constexpr int kPaths = 9;        // distinct paths per 128-row tile in the SGD kernel (N >= 16)
constexpr uint32_t kW1 = kU * kU * 4;        // one plane of W1 / W1^T (16 KB)
constexpr uint32_t kW0i = kU * kInd * 4;     // one plane of the W0 indicator block (2 KB)
constexpr uint32_t kH = kU * 128 * 4;        // one H1^T plane (32 KB)
constexpr uint32_t kG = 128 * 128 * 4;       // G^T stacked [hi rows 0..63; lo rows 64..127] (64 KB)
constexpr uint32_t kGlo = 8 * 1024;          // row 64 + o of a 128-row SW128 tile: 8 atoms past row o
constexpr int kBR = 32;                      // rows of the [indicators; path membership; 0] operand
constexpr uint32_t kB = kBR * 128 * 4;       // its single (exact) plane (16 KB)
constexpr int kSgdThreads = 512;             // 4 warpgroups x 16 columns
constexpr int kSlots = 5;                    // per-tile indicator / path-sum blocks kept in TMEM (N >= 128)
constexpr int kSlotsWide = 3;                // ... for N < 128 (up to 9 paths per tile: 32-column blocks)
// TMEM columns of the SGD kernel: D (layer-0 indicator part, then layer 1), A hi | lo
// (H1, then G2), gW1 [hi rows; lo rows] x 64, the indicator A operand (8 used), DB
// (the backward product G2 W1, then G1), the per-tile [128 x 16] (N >= 128) or
// [128 x 32] indicator / path-sum blocks, and act'(H1) of the tile in flight.
constexpr uint32_t kTD = 0, kTAh = 64, kTAl = 128, kTW1 = 192, kTInd = 256, kTB = 272, kTSlot = 336, kTDh = 448;
static_assert(kTSlot + 16 * kSlots <= kTDh && kTSlot + 32 * kSlotsWide <= kTDh, "TMEM columns");
__host__ __device__ constexpr int sgd_slots(int N) { return N >= 128 ? kSlots : kSlotsWide; }

constexpr size_t sgd_split_smem() {
    return 2ull * kH + kG + kB + 4ull * kW1 + 2ull * kW0i + 4ull * (kPaths * kQ + 2 * kPaths * kU + 4 * 128 + 2 * kU) +
           128 + 1024;
}

__device__ __forceinline__ void cta_sync() {
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
}

__device__ __forceinline__ uint8_t* align1k(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

__device__ __forceinline__ void sts(uint32_t addr, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

// Per-path part of layer 0 for the paths of a tile: P[p][o] = b0[o] + W0_y[o] . y_p,
// eight threads per output (strided partial sums, then a fixed shuffle tree).
__device__ __forceinline__ void path_projection8(const SplitArgs& a, const float* ysh, float* Psh, int np, int tid,
                                                 int nthreads) {
    const int sub = tid & 7;
    for (int i = tid >> 3; i < np * kU; i += nthreads >> 3) {
        const int p = i / kU, o = i % kU;
        const float* w = a.p32 + a.off0 + o * a.d + a.Cc;
        float s = 0.0f;
        for (int j = sub; j < a.q; j += 8) s = fmaf(__ldcg(w + j), ysh[p * kQ + j], s);
        s += __shfl_xor_sync(0xffffffffu, s, 4);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        if (sub == 0) Psh[p * kU + o] = __ldcg(a.vec + o) + s;
    }
}

// Row state of one 128-row tile for thread row r.
struct RowState {
    unsigned kfirst;  // first path of the tile
    int np;           // paths in the tile
    int p;            // this row's path (tile-local)
    unsigned ind;     // indicator bits 1{s_c <= i}
    double y;         // label
    bool live;
};

// Grid-wide barrier of the persistent SGD kernel (cooperative launch: every
// CTA is resident), split into arrive and wait so that work not depending on
// the other CTAs can run in between.  `count` is zeroed before the launch;
// barrier k of the launch waits for (k + 1) * gridDim.x arrivals.  The CTA
// barrier orders every thread's writes before thread 0's release (cumulative);
// the matching acquire is thread 0's poll.  A CTA that is never joined traps
// instead of hanging the GPU.
__device__ __forceinline__ void grid_arrive(unsigned* count) {
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
}
__device__ __forceinline__ void grid_wait(unsigned* count, unsigned target) {
    if (threadIdx.x == 0) {
        const long long t0 = clock64();
        unsigned v;
        while (true) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
            if (v >= target) break;
            if (clock64() - t0 > (1ll << 35)) __trap();
        }
    }
    __syncthreads();
}

// The global loads of a tile's row state (issued early, consumed later): the
// row's default steps and label, and this thread's share of the tile's path
// columns (element tid of np x q).
struct RowLoads {
    unsigned short st[kInd];
    double y;
    float yv;
};

// Element tid of the tile's np x q path columns (the layer-0 inputs of its paths).
__device__ __forceinline__ float path_col(const SplitArgs& a, long tile, int tid) {
    const unsigned row0 = static_cast<unsigned>(tile * 128), N = static_cast<unsigned>(a.N);
    const unsigned kfirst = row0 / N;
    const int np = static_cast<int>(min(row0 + 127u, static_cast<unsigned>(a.R - 1)) / N - kfirst + 1);
    return tid < np * a.q ? __ldg(a.yhat + static_cast<size_t>(kfirst + tid / a.q) * a.qp + tid % a.q) : 0.0f;
}

__device__ __forceinline__ RowLoads row_loads(const SplitArgs& a, long tile, int r, int tid, long b0, long b1) {
    RowLoads l;
    const unsigned row = static_cast<unsigned>(tile * 128) + r;
    const bool live = row >= b0 && row < b1;
#pragma unroll
    for (int c = 0; c < kInd; ++c)
        l.st[c] = (live && c < a.Cc) ? __ldg(a.steps + static_cast<size_t>(c + 1) * a.R + row) : 0xFFFF;
    l.y = live ? __ldg(a.y + row) : 0.0;
    l.yv = a.N >= 128 ? 0.0f : path_col(a, tile, tid);  // N >= 128: staged per step instead
    return l;
}

__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }


__device__ __forceinline__ RowState row_state(const SplitArgs& a, long tile, int r, const RowLoads& l, long b0,
                                              long b1) {
    RowState s;
    const unsigned row0 = static_cast<unsigned>(tile * 128), N = static_cast<unsigned>(a.N);
    s.kfirst = row0 / N;
    s.np = static_cast<int>(min(row0 + 127u, static_cast<unsigned>(a.R - 1)) / N - s.kfirst + 1);
    const unsigned row = row0 + r;
    s.live = row >= b0 && row < b1;
    s.p = s.live ? static_cast<int>(row / N - s.kfirst) : 0;
    s.ind = 0;
#pragma unroll
    for (int c = 0; c < kInd; ++c) s.ind |= (l.st[c] <= a.step ? 1u : 0u) << c;
    s.y = l.y;
    return s;
}

// Profiling: per-phase clock64 stamps of CTA 0's first tiles (SplitArgs::trace).
#define TRACE(k) \
    if (a.trace && blockIdx.x == 0 && tid == 0 && nt < 4) a.trace[nt * 16 + (k)] = clock64()
#define TRACE_FIX(k) \
    if (a.trace && blockIdx.x == 0 && tid == 0) a.trace[64 + (k)] = clock64()

template <int ACT>
__global__ void __launch_bounds__(kSgdThreads + 32, 1) k_sgd_split(SplitArgs a, long t_first, long n_tiles) {
    extern __shared__ uint8_t sm_raw[];
    uint8_t* sm = align1k(sm_raw);
    uint8_t* tH = sm;              // H1^T hi | lo planes, SW128 K-major, 64 x 128
    uint8_t* tG = tH + 2 * kH;     // G2^T, then G1^T, stacked hi | lo rows, 128 x 128
    uint8_t* tB = tG + kG;         // [indicators (8); path membership (9); 0] x 128, exact
    uint8_t* w1 = tB + kB;         // W1 hi | lo
    uint8_t* w1t = w1 + 2 * kW1;   // W1^T hi | lo
    uint8_t* w0b = w1t + 2 * kW1;  // W0 indicator columns [64 x 8] hi | lo (B operand)
    float* ysh = reinterpret_cast<float*>(w0b + 2 * kW0i);  // [p][kQ] y of a tile's paths
    float* Psh = ysh + kPaths * kQ;                        // [2][p][kU] layer-0 path parts, double buffered
    float* fsh = Psh + 2 * kPaths * kU;                    // [4][128] output-sum exchange
    float* vsh = fsh + 4 * 128;                            // b1 | w2
    // mbarriers: MMA completions 0 Z (D0), 1 F (F1), 2 X (B), 3 Y (gW1); 4 W (weights);
    // 5..8 operands ready for D0 / F1 / B + gW1 / slot + next D0 (one arrival per epilogue warp)
    // 9 slot MMAs done
    uint64_t* bar = reinterpret_cast<uint64_t*>(vsh + 2 * kU);
    uint32_t* tbase = reinterpret_cast<uint32_t*>(bar + 10);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool issuer = warp == kSgdThreads / 32;  // warp 16 issues every MMA; warps 0-15 are rows x columns
    const int r = tid & 127, hf = (tid >> 7) & 3, cb = hf * 16;
    if (tid == 0) {
        for (int i = 0; i < 5; ++i) tc::mbar_init(&bar[i], 1);
        for (int i = 5; i < 9; ++i) tc::mbar_init(&bar[i], kSgdThreads / 32);
        tc::mbar_init(&bar[9], 1);
        tc::fence_async_smem();
    }
    TRACE_FIX(0);
    if (warp == 0) tc::tmem_alloc(tbase, 512);
    for (int i = tid; i < kPaths * kQ; i += kSgdThreads + 32) ysh[i] = 0.0f;
    // transposed-store addresses of this thread: element (feature cb + q, batch row r)
    // of a SW128 K-major tile with R rows sits at base + x[q & 7] + (q >> 3) * 1024
    uint32_t xH[8], xG[8];
    {
        const uint32_t cr = (r & 31) >> 2;
        const uint32_t bH = tc::smem_u32(tH) + ((r >> 5) * (kU / 8) + cb / 8) * 1024u + (r & 3) * 4u;
        const uint32_t bG = tc::smem_u32(tG) + ((r >> 5) * (128 / 8) + cb / 8) * 1024u + (r & 3) * 4u;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            xH[k] = bH + k * 128u + ((cr ^ k) << 4);
            xG[k] = bG + k * 128u + ((cr ^ k) << 4);
        }
    }
    // Persistent mode (a.fuse): a.nsteps SGD steps over consecutive batches of a.bs
    // rows from a.b0, the optimizer fused behind two grid barriers per step.
    const int nsteps = a.fuse ? a.nsteps : 1;
    // the first tile's row loads do not depend on the optimizer: before the dependency wait
    const long b1_0 = a.fuse ? a.b0 + a.bs : a.b1;
    // (in persistent mode the next step's are loaded during the optimizer's last barrier)
    RowLoads lfirst = (!issuer && blockIdx.x < n_tiles) ? row_loads(a, t_first + blockIdx.x, r, tid, a.b0, b1_0)
                                                        : RowLoads{};
    // N >= 128 (a tile holds at most 2 paths): the per-path columns of every tile of
    // this CTA's step, staged once per step as ys2 [2 * tile + p][kQ]
    const bool pre = a.N >= 128;
    float* ys2 = Psh + 2 * kSlots * kU;
    auto load_ys2 = [&](long tf_, long t_end_) {
        const int ntl = static_cast<int>((t_end_ - (tf_ + blockIdx.x) + gridDim.x - 1) / gridDim.x);
        for (int i = tid; i < ntl * 2 * kQ; i += kSgdThreads) {
            const int k = i / (2 * kQ), p = (i / kQ) % 2, j = i % kQ;
            const unsigned row0 = static_cast<unsigned>((tf_ + blockIdx.x + static_cast<long>(k) * gridDim.x) * 128);
            const unsigned kf = row0 / static_cast<unsigned>(a.N);
            const bool in = j < a.q && kf + p < static_cast<unsigned>(a.M);
            ys2[i] = in ? __ldg(a.yhat + static_cast<size_t>(kf + p) * a.qp + j) : 0.0f;
        }
    };
    cta_sync();
    const uint32_t tm = *tbase;
    const uint32_t lb = static_cast<uint32_t>((warp & 3) * 32) << 16;
    pdl_wait();  // the optimizer's parameters and weight image
    const uint32_t id128 = tc::idesc_tf32(128, kU, 0, 0);
    uint32_t ph[4] = {0, 0, 0, 0}, rph[4] = {0, 0, 0, 0}, sph = 0;  // sph: slot-MMA completions (barrier 9)
    unsigned gsyncs = 0;
    for (int step = 0; step < nsteps; ++step) {
    const long sb0 = a.fuse ? a.b0 + step * a.bs : a.b0, sb1 = a.fuse ? sb0 + a.bs : a.b1;
    const long tf = sb0 / 128, t_end = (sb1 - 1) / 128 + 1;
    TRACE_FIX(16);
    if (tid == 0) {
        if (step > 0) asm volatile("fence.proxy.async.global;" ::: "memory");  // the image the optimizer wrote
        tc::mbar_expect_tx(&bar[4], 4 * kW1);
        tc::bulk_g2s(w1, a.w1img, 4 * kW1, &bar[4]);
    }
    double loss = 0.0, dmu = 0.0;
    float gb2 = 0.0f, acc_w2 = 0.0f, acc_b1 = 0.0f;
    int nt = 0;

    if (issuer) {
        // ================= MMA issue (one lane), paced by the epilogue warps' ready barriers.
        // Per tile n: B(n), the next tile's D0, gW1(n), the next tile's F1, slot(n) -- so the
        // next tile's layer 0 (epilogue) overlaps gW1(n) and its F1 follows gW1 directly.
        auto wait_ready = [&](int k) {
            tc::mbar_wait(&bar[5 + k], rph[k]);
            rph[k] ^= 1;
            tc::fence_after_sync();
        };
        auto issue_d0 = [&]() {  // D0 = ind W0_ind^T (exact A: two MMAs), commit Z
            const tc::Operand B = tc::kmajor(w0b, kW0i, kU);
            tc::mma_tf32_ts(tm + kTD, tm + kTInd, B.desc(0, 0), id128, 0);
            tc::mma_tf32_ts(tm + kTD, tm + kTInd, B.desc(1, 0), id128, 1);
            tc::commit(&bar[0]);
        };
        auto issue_f1 = [&]() {  // F1: D = H1 W1^T, H1 from tensor memory; commit F
            tc::gemm3_ts(tm + kTD, tm + kTAh, tm + kTAl, tc::kmajor(w1, kW1, kU), kU, id128, 0);
            tc::commit(&bar[1]);
        };
        tc::mbar_wait(&bar[4], step & 1);  // W1 / W1^T in shared memory
        long t = tf + blockIdx.x;
        if (t < t_end) {
            wait_ready(0);
            if (lane == 0) issue_d0();
            wait_ready(1);
            if (lane == 0) issue_f1();
        }
        const uint32_t sw = static_cast<uint32_t>(pre ? 16 : 32);
        for (int n = 0; t < t_end; t += gridDim.x, ++n) {
            const bool more = t + gridDim.x < t_end;
            if (more) {  // the next tile's rows (default steps, labels) into L2 while this tile runs
                const unsigned row0 = static_cast<unsigned>((t + gridDim.x) * 128);
                if (lane < kInd && lane < a.Cc) {  // 256 B of default steps per name: two lines
                    const uint16_t* p = a.steps + static_cast<size_t>(lane + 1) * a.R + row0;
                    prefetch_l2(p);
                    prefetch_l2(p + 64);
                }
                if (lane >= 16 && lane < 24) prefetch_l2(a.y + row0 + 16 * (lane - 16));  // 1 KB of labels
            }
            wait_ready(2);
            if (lane == 0) {  // ---- B: DB = G2 W1 (the W1^T tile), G2 from tensor memory; commit X
                tc::gemm3_ts(tm + kTB, tm + kTAh, tm + kTAl, tc::kmajor(w1t, kW1, kU), kU, id128, 0);
                tc::commit(&bar[2]);
            }
            if (more) {
                wait_ready(0);
                if (lane == 0) issue_d0();  // the next tile's D0 (the epilogue's next layer 0 waits on it)
            }
            if (lane == 0) {
                // ---- gW1 += [G2^T hi; G2^T lo] (H1^T hi + H1^T lo): M = 128, two MMAs per K step; commit Y
                const tc::OperandSW A{tc::smem_u32(tG), 0, 128, 0};
                const tc::OperandSW Bh{tc::smem_u32(tH), 0, kU, 0}, Bl{tc::smem_u32(tH) + kH, 0, kU, 0};
                const uint32_t id = tc::idesc_tf32(128, kU, 0, 0);
#pragma unroll 1
                for (int ks = 0; ks < 16; ++ks) {
                    tc::mma_tf32(tm + kTW1, A.desc(0, ks), Bh.desc(0, ks), id, (ks > 0 || n > 0) ? 1 : 0);
                    tc::mma_tf32(tm + kTW1, A.desc(0, ks), Bl.desc(0, ks), id, 1);
                }
                tc::commit(&bar[3]);
            }
            if (more) {
                wait_ready(1);
                if (lane == 0) issue_f1();  // the next tile's F1, queued behind gW1(n)
            }
            wait_ready(3);
            if (lane == 0) {
                // ---- slot = [G1^T hi; G1^T lo] [ind; member] (exact B, M = 128): read at the end; commit S
                const tc::OperandSW A{tc::smem_u32(tG), 0, 128, 0}, Bm{tc::smem_u32(tB), 0, kBR, 0};
                const uint32_t id = tc::idesc_tf32(128, sw, 0, 0), slot = tm + kTSlot + sw * n;
#pragma unroll 1
                for (int ks = 0; ks < 16; ++ks) tc::mma_tf32(slot, A.desc(0, ks), Bm.desc(0, ks), id, ks > 0 ? 1 : 0);
                tc::commit(&bar[9]);
            }
            nt = n + 1;
        }
        __syncwarp();
    } else {
        // ================= epilogue warps: 128 rows x 4 column groups of 16
        for (int i = tid; i < kInd * kU; i += kSgdThreads) {
            const int o = i / kInd, c = i % kInd;
            tc::put_split(w0b, kW0i, o, c, kU, c < a.Cc ? __ldcg(a.p32 + a.off0 + o * a.d + c) : 0.0f);
        }
        const float b2 = __ldcg(a.vec + 192);
        const double mu = __ldcg(a.mu64), two_nb = 2.0 / a.nb;
        if (tid < 2 * kU) vsh[tid] = __ldcg(a.vec + 64 + tid);  // b1 | w2
        const float* b1v = vsh + cb;
        const float* w2v = vsh + kU + cb;
        auto epi_sync = [&]() { asm volatile("bar.sync 1, %0;" ::"n"(kSgdThreads) : "memory"); };
        auto wait_done = [&](int b) {
            tc::mbar_wait(&bar[b], ph[b]);
            ph[b] ^= 1;
            tc::fence_after_sync();
        };
        auto ready = [&](int k) {  // this warp's operand writes for the next MMAs are complete
            tc::tmem_wait_st();
            tc::fence_async_smem();
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&bar[5 + k])) : "memory");
        };
        // layer-0 inputs of a tile: its paths' y, P into Psh[buf], the indicator A operand
        // N >= 128 (a tile holds at most 2 paths): the layer-0 path parts of every
        // tile of this CTA's step at once, Psh [2 * tile + p][64], W0_y rows loaded once
        if (pre) {
            const int ntl = static_cast<int>((t_end - (tf + blockIdx.x) + gridDim.x - 1) / gridDim.x);
            if (step == 0) load_ys2(tf, t_end);
            const int o = tid >> 3, sub = tid & 7;
            float w[kQ / 8];
#pragma unroll
            for (int m = 0; m < kQ / 8; ++m)
                w[m] = sub + 8 * m < a.q ? __ldcg(a.p32 + a.off0 + o * a.d + a.Cc + sub + 8 * m) : 0.0f;
            const float b0o = __ldcg(a.vec + o);
            epi_sync();
            for (int qi = 0; qi < 2 * ntl; ++qi) {
                float acc = 0.0f;
#pragma unroll
                for (int m = 0; m < kQ / 8; ++m) acc = fmaf(w[m], ys2[qi * kQ + sub + 8 * m], acc);
                acc += __shfl_xor_sync(0xffffffffu, acc, 4);
                acc += __shfl_xor_sync(0xffffffffu, acc, 2);
                acc += __shfl_xor_sync(0xffffffffu, acc, 1);
                if (sub == 0) Psh[qi * kU + o] = b0o + acc;
            }
            TRACE_FIX(17);
        }
        auto stage_tile = [&](const RowState& st, float yv, int buf) {
            if (!pre && tid < st.np * a.q) ysh[(tid / a.q) * kQ + tid % a.q] = yv;
            if (hf == 0) {
                float iv[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) iv[c] = ((st.ind >> c) & 1u) ? 1.0f : 0.0f;
                tc::tmem_st8(tm + lb + kTInd, iv);
            }
            if (!pre) {
                epi_sync();
                path_projection8(a, ysh, Psh + buf * kPaths * kU, st.np, tid, kSgdThreads);
            }
        };
        // Layer 0 of a tile -> H1: hi | lo into tensor memory (the A operand of F1),
        // act'(H1) into tensor memory; the transposed H1^T (the gW1 operand) is written
        // separately (store_h1t), once the previous tile's gW1 has read its buffer.
        auto layer0 = [&](const RowState& st, const float* Pt) {
            float z[16], hi[16], lo[16], dh[16];
            const float* P = Pt + st.p * kU + cb;
            tc::tmem_ld16(tm + lb + kTD + cb, z);
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const float h = act_f<ACT>(z[q] + P[q]);
                hi[q] = tc::tf32_rna(h);
                lo[q] = h - hi[q];
                dh[q] = act_d<ACT>(h);
            }
            tc::tmem_st16(tm + lb + kTAh + cb, hi);
            tc::tmem_st16(tm + lb + kTAl + cb, lo);
            tc::tmem_st16(tm + lb + kTDh + cb, dh);
        };
        auto store_h1t = [&]() {  // H1^T hi | lo planes from the A operand in tensor memory
            float hi[16], lo[16];
            tc::tmem_ld16(tm + lb + kTAh + cb, hi);
            tc::tmem_ld16(tm + lb + kTAl + cb, lo);
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                sts(xH[q & 7] + (q >> 3) * 1024u, hi[q]);
                sts(xH[q & 7] + (q >> 3) * 1024u + kH, lo[q]);
            }
        };
        auto path_parts = [&](int k, int pbuf) {  // P of tile k of this step (pre) / the staged buffer
            return pre ? Psh + 2 * k * kU : Psh + pbuf * kPaths * kU;
        };
        int buf = 0;
        long tile = tf + blockIdx.x;
        RowState cur{};
        if (tile < t_end) {  // the step's first tile: stage, D0, layer 0, F1
            cur = row_state(a, tile, r, lfirst, sb0, sb1);
            stage_tile(cur, lfirst.yv, 0);
            ready(0);
            epi_sync();  // Psh of the first tile complete
            wait_done(0);
            layer0(cur, path_parts(0, 0));
            store_h1t();
            ready(1);
        }
        TRACE_FIX(1);
        TRACE_FIX(2);
        for (; tile < t_end; tile += gridDim.x, ++nt, buf ^= 1) {
            const bool more = tile + gridDim.x < t_end;
            TRACE(0);
            wait_done(1);  // F1 of this tile
            TRACE(1);
            // ---- epilogue 2: H2, f, residual, G2 (TMEM A for B, G2^T for gW1), this tile's
            // rows of the slot operand [ind; member]
            float h2[16];
            tc::tmem_ld16(tm + lb + kTD + cb, h2);
            float fp = 0.0f;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                h2[j] = act_f<ACT>(h2[j] + b1v[j]);
                fp = fmaf(h2[j], w2v[j], fp);
            }
            fsh[hf * 128 + r] = fp;
            epi_sync();
            const float f = b2 + ((fsh[r] + fsh[128 + r]) + (fsh[256 + r] + fsh[384 + r]));
            float dd = 0.0f;
            if (cur.live) {
                const double pr = ((a.head && f < 0.0f) ? 0.0 : static_cast<double>(f)) + mu;
                const double res = pr - cur.y;
                const double dm = res * two_nb;
                if (hf == 0) {
                    loss += res * res;
                    dmu += dm;
                }
                dd = static_cast<float>(dm);
                if (a.head && !(f > 0.0f)) dd = 0.0f;
            }
            if (hf == 0) gb2 += dd;
            {
                float g[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) g[j] = dd * h2[j];
                acc_w2 += bfly_sum<16>(g, lane);  // lane: column cb + lane % 16 over the warp's rows
            }
            TRACE(2);
            if (nt > 0) {  // the previous tile's slot MMAs have read G1^T and [ind; member]
                tc::mbar_wait(&bar[9], sph);
                sph ^= 1;
                tc::fence_after_sync();
            }
#pragma unroll
            for (int n = 0; n < kBR / 4; ++n) {
                const int br = hf * (kBR / 4) + n;
                float v = 0.0f;
                if (br < kInd) v = ((cur.ind >> br) & 1u) ? 1.0f : 0.0f;
                else if (br < kInd + kPaths) v = (cur.live && cur.p == br - kInd) ? 1.0f : 0.0f;
                *reinterpret_cast<float*>(tB + tc::sw_off(br, r, kBR)) = v;
            }
            {
                float gv[16], hi[16], lo[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    gv[q] = dd * w2v[q] * act_d<ACT>(h2[q]);
                    hi[q] = tc::tf32_rna(gv[q]);
                    lo[q] = gv[q] - hi[q];
                    sts(xG[q & 7] + (q >> 3) * 1024u, hi[q]);
                    sts(xG[q & 7] + (q >> 3) * 1024u + kGlo, lo[q]);
                }
                tc::tmem_st16(tm + lb + kTAh + cb, hi);
                tc::tmem_st16(tm + lb + kTAl + cb, lo);
                acc_b1 += bfly_sum<16>(gv, lane);  // gb1: column sums of G2
            }
            ready(2);
            TRACE(3);
            RowState nxt{};
            if (more) {  // the next tile's layer-0 inputs (indicator operand, P), under B; then its D0
                const RowLoads ln = row_loads(a, tile + gridDim.x, r, tid, sb0, sb1);
                nxt = row_state(a, tile + gridDim.x, r, ln, sb0, sb1);
                stage_tile(nxt, ln.yv, buf ^ 1);
                ready(0);
            }
            TRACE(4);
            wait_done(2);  // B: DB = G2 W1
            TRACE(5);
            {  // ---- G1 = DB act'(H1), kept in DB
                float g1[16], dh[16];
                tc::tmem_ld16(tm + lb + kTB + cb, g1);
                tc::tmem_ld16(tm + lb + kTDh + cb, dh);
#pragma unroll
                for (int q = 0; q < 16; ++q) g1[q] *= dh[q];
                tc::tmem_st16(tm + lb + kTB + cb, g1);
            }
            TRACE(6);
            if (more) {  // ---- the next tile's layer 0, while gW1(n) runs
                if (!pre) epi_sync();  // its staged P complete
                wait_done(0);
                layer0(nxt, path_parts(nt + 1, buf ^ 1));
                ready(1);
            }
            TRACE(7);
            wait_done(3);  // gW1(n): G2^T and H1^T read
            TRACE(8);
            {  // ---- G1^T for the slot MMAs, then the next tile's H1^T
                float g1[16];
                tc::tmem_ld16(tm + lb + kTB + cb, g1);
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const float hi = tc::tf32_rna(g1[q]);
                    sts(xG[q & 7] + (q >> 3) * 1024u, hi);
                    sts(xG[q & 7] + (q >> 3) * 1024u + kGlo, g1[q] - hi);
                }
            }
            if (more) store_h1t();
            ready(3);
            TRACE(9);
            TRACE(10);
            cur = nxt;
        }
        if (nt > 0) {  // the last slot MMAs (and with them every MMA of the step)
            tc::mbar_wait(&bar[9], sph);
            sph ^= 1;
            tc::fence_after_sync();
        }
    }
    __syncthreads();
    TRACE_FIX(3);
    TRACE_FIX(4);

    // ---- this CTA's partial row of the gradient (every parameter); scratch in tH / tG
    // partial rows: stride P, padded to 16 bytes in persistent mode (16-byte gathers)
    const int gld = a.fuse ? (a.P + 3) & ~3 : a.P;
    float* gout = a.gpart + static_cast<size_t>(blockIdx.x) * gld;
    constexpr int L1 = kU + 1;                 // padded rows: conflict-free column stores
    float* s1 = reinterpret_cast<float*>(tH);  // [128][L1] gW1 rows: hi part, lo part
    float* s2 = reinterpret_cast<float*>(tG);  // [128][kInd + 1 + kQ + 1] gW0 rows: hi part, lo part
    if (warp < 4) {
#pragma unroll
        for (int c = 0; c < kU; c += 16) {
            float v[16];
            tc::tmem_ld16(tm + lb + kTW1 + c, v);
#pragma unroll
            for (int q = 0; q < 16; ++q) s1[r * L1 + c + q] = v[q];
        }
    }
    TRACE_FIX(5);
    float* part = fsh;                                      // [warp][32] w2, then b1 partials
    double* red = reinterpret_cast<double*>(Psh);          // [3][16]
    if (!issuer) part[warp * 32 + lane] = acc_w2;
    loss = warp_sum(loss);
    dmu = warp_sum(dmu);
    const float gb2w = warp_sum(gb2);
    if (lane == 0 && !issuer) {
        red[warp] = loss;
        red[16 + warp] = dmu;
        red[32 + warp] = gb2w;
    }
    __syncthreads();
    if (tid < kU) {  // column tid: warpgroup tid / 16, lane tid % 16 of its four warps
        const int w0q = (tid / 16) * 4, c = tid % 16;
        gout[a.off2 + tid] = part[(w0q + 0) * 32 + c] + part[(w0q + 1) * 32 + c] + part[(w0q + 2) * 32 + c] +
                             part[(w0q + 3) * 32 + c];
    }
    if (tid == 0) {  // warpgroup 0 holds the per-row terms
        a.lpart[blockIdx.x] = red[0] + red[1] + red[2] + red[3];
        gout[a.P - 1] = static_cast<float>(red[16] + red[17] + red[18] + red[19]);
        gout[a.off2 + kU] = static_cast<float>(red[32] + red[33] + red[34] + red[35]);
    }
    __syncthreads();
    TRACE_FIX(8);
    if (!issuer) part[warp * 32 + lane] = acc_b1;
    __syncthreads();
    if (tid < kU) {
        const int w0q = (tid / 16) * 4, c = tid % 16;
        gout[a.off1 + kU * kU + tid] = part[(w0q + 0) * 32 + c] + part[(w0q + 1) * 32 + c] +
                                       part[(w0q + 2) * 32 + c] + part[(w0q + 3) * 32 + c];
    }
    TRACE_FIX(9);
    // gW1[o][i] = hi-row + lo-row of the stacked accumulator
    for (int i = tid; i < kU * kU; i += kSgdThreads + 32) {
        const int o = i / kU, c = i % kU;
        gout[a.off1 + i] = nt == 0 ? 0.0f : s1[o * L1 + c] + s1[(kU + o) * L1 + c];
    }
    TRACE_FIX(10);
    // gW0 from the slots: accumulator row r' (TMEM lane r', warps 0-3) is output
    // row r' % 64, hi part for r' < 64, lo part above.  Per slot (tile order):
    // the indicator columns, and per path (path order) s_p -> b0 and s_p y_p.
    int* snp = reinterpret_cast<int*>(red + 48);                          // [kSlots] paths per slot
    // per-path columns of each slot's paths: ys2 when staged per step, else loaded here
    float* yh = pre ? ys2 : reinterpret_cast<float*>(tH + 128 * (kU + 1) * 4 + 64);  // [slot][ystr][kQ]
    const int ystr = pre ? 2 : kPaths;
    if (tid < nt) {
        const unsigned row0 = static_cast<unsigned>((tf + blockIdx.x + static_cast<long>(tid) * gridDim.x) * 128);
        const unsigned N = static_cast<unsigned>(a.N);
        snp[tid] = static_cast<int>(min(row0 + 127u, static_cast<unsigned>(a.R - 1)) / N - row0 / N + 1);
    }
    if (!pre) {
        for (int i = tid; i < nt * kPaths * kQ; i += kSgdThreads + 32) {
            const int s = i / (kPaths * kQ), p = (i / kQ) % kPaths, j = i % kQ;
            const unsigned row0 = static_cast<unsigned>((tf + blockIdx.x + static_cast<long>(s) * gridDim.x) * 128);
            const unsigned kf = row0 / static_cast<unsigned>(a.N);
            const bool in = j < a.q && kf + p < static_cast<unsigned>(a.M);
            yh[i] = in ? __ldg(a.yhat + static_cast<size_t>(kf + p) * a.qp + j) : 0.0f;
        }
    }
    __syncthreads();
    TRACE_FIX(11);
    // Slots over the four warpgroups by columns: warpgroup g accumulates the y columns
    // [12 g, 12 g + 12) over every slot (and warpgroup 0 the indicator columns and b0),
    // each element summed over slots and paths in order.
    constexpr int LW = kInd + 1 + kQ + 1;  // s2 row: indicators, b0, y columns (padded)
    constexpr int kQg = kQ / 4;
    if (!issuer) {
        const int wg = warp >> 2;
        float acc_i[kInd], acc_y[kQg], acc_b0 = 0.0f;
#pragma unroll
        for (int c = 0; c < kInd; ++c) acc_i[c] = 0.0f;
#pragma unroll
        for (int j = 0; j < kQg; ++j) acc_y[j] = 0.0f;
        for (int sl = 0; sl < nt; ++sl) {
            float v[32];
            const uint32_t sw = pre ? 16u : 32u;
            tc::tmem_ld16(tm + lb + kTSlot + sw * sl, v);
            if (pre) {
#pragma unroll
                for (int c = 16; c < 32; ++c) v[c] = 0.0f;
            } else {
                tc::tmem_ld16(tm + lb + kTSlot + sw * sl + 16, v + 16);
            }
#pragma unroll
            for (int c = 0; c < kInd; ++c) acc_i[c] += v[c];
            const int np = snp[sl];
#pragma unroll
            for (int p = 0; p < kPaths; ++p) {
                if (p >= np) break;
                const float sp = v[kInd + p];
                acc_b0 += sp;
                const float* y = yh + (sl * ystr + p) * kQ + wg * kQg;
#pragma unroll
                for (int j = 0; j < kQg; ++j) acc_y[j] = fmaf(sp, y[j], acc_y[j]);
            }
        }
        float* row = s2 + r * LW;
        if (wg == 0) {
#pragma unroll
            for (int c = 0; c < kInd; ++c) row[c] = acc_i[c];
            row[kInd] = acc_b0;
        }
#pragma unroll
        for (int j = 0; j < kQg; ++j) row[kInd + 1 + wg * kQg + j] = acc_y[j];
    }
    __syncthreads();
    TRACE_FIX(12);
    if (tid < kSgdThreads) {  // output row o = tid / 8, columns c = tid % 8, +8, ...
        const int o = tid >> 3, W = kInd + 1 + a.q;
        for (int c = tid & 7; c < W; c += 8) {
            const float v = s2[o * LW + c] + s2[(kU + o) * LW + c];
            if (c < kInd) {
                if (c < a.Cc) gout[a.off0 + o * a.d + c] = v;
            } else if (c == kInd) {
                gout[a.off0 + kU * a.d + o] = v;
            } else {
                gout[a.off0 + o * a.d + a.Cc + (c - kInd - 1)] = v;
            }
        }
    }
    TRACE_FIX(6);
    if (a.fuse) {
        // ---- the optimizer, fused: every CTA's partial row is written; CTA c reduces
        // parameters [c per, (c+1) per) over the rows in fixed order, updates them
        // (regressor.cpp:236-261) and refreshes the weight image; then every CTA
        // reloads the weights for the next step
        const int P = a.P, G = gridDim.x;
        const int per = ((P + G - 1) / G + 3) & ~3, i0 = blockIdx.x * per, cnt = min(P, i0 + per) - i0;
        const double c1 = __ldcg(a.c12 + 2 * step), c2 = __ldcg(a.c12 + 2 * step + 1);
        // this CTA's slice of the optimizer state: only this CTA updates it, so it is
        // read before the barrier
        double w_own = 0.0, m_own = 0.0, v_own = 0.0;
        if (tid < cnt) {
            w_own = __ldcg(a.p64w + i0 + tid);
            m_own = __ldcg(a.m + i0 + tid);
            v_own = __ldcg(a.v + i0 + tid);
        }
        grid_arrive(a.gbar);
        grid_wait(a.gbar, ++gsyncs * G);
        TRACE_FIX(13);
        double lsum = 0.0;  // the batch loss (CTA 0's MMA-issue warp), consumed after the update
        if (blockIdx.x == 0 && issuer)
            for (int c = lane; c < G; c += 32) lsum += __ldcg(a.lpart + c);
        ImgArgs im;
        im.img = a.img;
        im.U = kU;
        im.d = a.d;
        im.dp = a.dp;
        im.off0 = a.off0;
        im.off1 = a.off1;
        im.off2 = a.off2;
        if (cnt > 0) {
            // the slice of every partial row into shared memory (16-byte loads, four in
            // flight per thread), then summed in FP64: ng groups of consecutive rows, the
            // group sums in group order
            float* rows = reinterpret_cast<float*>(tH);  // [G][per]
            const int nq = (cnt + 3) >> 2, nall = G * nq;
            for (int i = tid; i < nall; i += 4 * (kSgdThreads + 32)) {
                float4 v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int k = i + u * (kSgdThreads + 32), c = k / nq, qq = k % nq;
                    if (k < nall) v[u] = __ldcg(reinterpret_cast<const float4*>(a.gpart + static_cast<size_t>(c) * gld + i0) + qq);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int k = i + u * (kSgdThreads + 32), c = k / nq, qq = k % nq;
                    if (k < nall) *reinterpret_cast<float4*>(rows + c * per + 4 * qq) = v[u];
                }
            }
            __syncthreads();
            TRACE_FIX(18);
            const int ng = min(8, (kSgdThreads + 32) / per);
            double* part = reinterpret_cast<double*>(tG);  // [ng][per]
            if (tid < ng * per) {
                const int j = tid % per, k = tid / per, ca = k * G / ng, ce = (k + 1) * G / ng;
                double g = 0.0;
                for (int c = ca; c < ce; ++c) g += static_cast<double>(rows[c * per + j]);
                part[k * per + j] = g;
            }
            __syncthreads();
            TRACE_FIX(19);
            if (tid < cnt) {  // Adam / SGD (regressor.cpp:236-261) on the prefetched state
                const int i = i0 + tid;
                double g = 0.0;
                for (int k = 0; k < ng; ++k) g += part[k * per + tid];
                double wv = w_own;
                if (a.adam) {
                    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
                    const double mi = b1 * m_own + (1.0 - b1) * g;
                    const double vi = b2 * v_own + (1.0 - b2) * g * g;
                    a.m[i] = mi;
                    a.v[i] = vi;
                    wv -= a.lr * (mi / c1) / (sqrt(vi / c2) + eps);
                } else {
                    wv -= a.lr * g;
                }
                a.p64w[i] = wv;
                a.p32w[i] = static_cast<float>(wv);
                img_store(im, P, i, static_cast<float>(wv));
            }
        }
        if (blockIdx.x == 0 && issuer) {  // the batch loss must stay finite (regressor.cpp:291-293)
            const double l = warp_sum(lsum);
            if (lane == 0 && !isfinite(l / a.nb)) atomicExch(a.nonfinite, 1);
        }
        TRACE_FIX(14);
        grid_arrive(a.gbar);
        ++gsyncs;
        {  // the next step's loads that do not need the new weights (lfirst is
           // assigned on every path: the previous value is dead during the tiles)
            const long nb0 = sb0 + a.bs, ntf = nb0 / 128, nt_end = (nb0 + a.bs - 1) / 128 + 1;
            const bool more = step + 1 < nsteps && !issuer;
            lfirst = (more && ntf + blockIdx.x < nt_end) ? row_loads(a, ntf + blockIdx.x, r, tid, nb0, nb0 + a.bs)
                                                        : RowLoads{};
            if (more && pre) load_ys2(ntf, nt_end);
        }
        grid_wait(a.gbar, gsyncs * G);
        TRACE_FIX(15);
    }
    }  // step
    tc::fence_before_sync();
    __syncthreads();
    TRACE_FIX(7);
    if (warp == 0) tc::tmem_dealloc(tm, 512);
}

// Layer-0 path parts of every path for an evaluation (W0 fixed during it):
// Pg[k][o] = b0[o] + W0_y[o] . y_k.  A CTA takes 64 paths: thread (o, g) keeps
// W0_y row o in registers and walks paths g, g + 4, ... of the block (the y
// rows staged in shared memory), sequential FMA order over j as elsewhere.
constexpr int kPjPaths = 64;
__global__ void __launch_bounds__(256) k_path_proj(SplitArgs a, float* Pg) {
    __shared__ float ys[kPjPaths * kQ];
    const long k0 = static_cast<long>(blockIdx.x) * kPjPaths;
    const int np = static_cast<int>(min(static_cast<long>(kPjPaths), a.M - k0));
    for (int i = threadIdx.x; i < np * a.q; i += blockDim.x)
        ys[(i / a.q) * kQ + i % a.q] = __ldg(a.yhat + (k0 + i / a.q) * a.qp + i % a.q);
    const int o = threadIdx.x & (kU - 1), g = threadIdx.x / kU;
    float w[kQ];
#pragma unroll
    for (int j = 0; j < kQ; ++j) w[j] = j < a.q ? __ldg(a.p32 + a.off0 + o * a.d + a.Cc + j) : 0.0f;
    const float b0 = __ldg(a.vec + o);
    __syncthreads();
    for (int p = g; p < np; p += 256 / kU) {
        float s = 0.0f;
#pragma unroll
        for (int j = 0; j < kQ; ++j)
            if (j < a.q) s = fmaf(w[j], ys[p * kQ + j], s);
        Pg[(k0 + p) * kU + o] = b0 + s;
    }
}

// ---------------------------------------------------------------- evaluation
// k_eval_split: one CTA per SM, 16 epilogue warps (128 rows x 4 groups of 16
// columns) and an MMA-issue warp, two tiles in flight: while F1 of tile n
// runs on the tensor cores, the epilogue finishes tile n-1 (H2, f, outputs)
// and prepares tile n+1 (default steps, path columns, P, the indicator
// operand whose D0 MMA follows).  Per TMEM buffer b = n & 1: D (D0, then F1's
// accumulator), H1 hi | lo (A operand), indicators.
constexpr int kEvThreads = 512;
constexpr uint32_t kEvBuf = 256;  // TMEM columns per buffer: D 0, A hi 64, A lo 128, indicators 192
constexpr size_t eval_split_smem() { return 2ull * kW1 + 2ull * kW0i + 4ull * (4 * 128 + 2 * kU) + 128 + 128; }

template <int ACT>
__global__ void __launch_bounds__(kEvThreads + 32, 1) k_eval_split(SplitArgs a, long t_first, long n_tiles) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* w1 = sm;                                        // W1 hi | lo
    uint8_t* w0b = w1 + 2 * kW1;                             // W0 indicator columns [64 x 8] hi | lo
    float* fsh = reinterpret_cast<float*>(w0b + 2 * kW0i);  // [4][128]
    float* vsh = fsh + 4 * 128;                              // b1 | w2
    // mbarriers: 0/1 D0 done, 2/3 F1 done, 4/5 D0 operands ready, 6/7 F1 operands ready, 8 weights
    uint64_t* bar = reinterpret_cast<uint64_t*>(vsh + 2 * kU);
    uint32_t* tbase = reinterpret_cast<uint32_t*>(bar + 9);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool issuer = warp == kEvThreads / 32;
    const int r = tid & 127, hf = (tid >> 7) & 3, cb = hf * 16;
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) tc::mbar_init(&bar[i], 1);
        for (int i = 4; i < 8; ++i) tc::mbar_init(&bar[i], kEvThreads / 32);
        tc::mbar_init(&bar[8], 1);
        tc::fence_async_smem();
    }
    if (warp == 0) tc::tmem_alloc(tbase, 512);
    cta_sync();
    const uint32_t tm = *tbase;
    const uint32_t lb = static_cast<uint32_t>((warp & 3) * 32) << 16;
    pdl_wait();
    if (tid == 0) {
        tc::mbar_expect_tx(&bar[8], 2 * kW1);
        tc::bulk_g2s(w1, a.w1img, 2 * kW1, &bar[8]);
    }
    const uint32_t id128 = tc::idesc_tf32(128, kU, 0, 0);
    const int nt = n_tiles > blockIdx.x ? static_cast<int>((n_tiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
    double loss = 0.0, mn = INFINITY;
    if (issuer) {
        uint32_t rph[4] = {0, 0, 0, 0};
        auto wait_ready = [&](int k) {
            tc::mbar_wait(&bar[4 + k], rph[k]);
            rph[k] ^= 1;
            tc::fence_after_sync();
        };
        auto d0 = [&](int b) {
            const tc::Operand B = tc::kmajor(w0b, kW0i, kU);
            const uint32_t base = tm + b * kEvBuf;
            tc::mma_tf32_ts(base, base + 192, B.desc(0, 0), id128, 0);
            tc::mma_tf32_ts(base, base + 192, B.desc(1, 0), id128, 1);
            tc::commit(&bar[b]);
        };
        tc::mbar_wait(&bar[8], 0);
        if (nt > 0) {
            wait_ready(0);
            if (lane == 0) d0(0);
        }
        for (int n = 0; n < nt; ++n) {
            const int b = n & 1;
            wait_ready(2 + b);
            if (lane == 0) {
                const uint32_t base = tm + b * kEvBuf;
                tc::gemm3_ts(base, base + 64, base + 128, tc::kmajor(w1, kW1, kU), kU, id128, 0);
                tc::commit(&bar[2 + b]);
            }
            if (n + 1 < nt) {
                wait_ready(b ^ 1);
                if (lane == 0) d0(b ^ 1);
            }
        }
        __syncwarp();
    } else {
        for (int i = tid; i < kInd * kU; i += kEvThreads) {
            const int o = i / kInd, c = i % kInd;
            tc::put_split(w0b, kW0i, o, c, kU, c < a.Cc ? a.p32[a.off0 + o * a.d + c] : 0.0f);
        }
        if (tid < 2 * kU) vsh[tid] = __ldg(a.vec + 64 + tid);  // b1 | w2
        const float b2 = __ldg(a.vec + 192);
        const double mu = a.mu64[0];
        uint32_t ph[4] = {0, 0, 0, 0};
        auto epi_sync = [&]() { asm volatile("bar.sync 1, %0;" ::"n"(kEvThreads) : "memory"); };
        auto wait_done = [&](int k) {
            tc::mbar_wait(&bar[k], ph[k]);
            ph[k] ^= 1;
            tc::fence_after_sync();
        };
        auto ready = [&](int k) {
            tc::tmem_wait_st();
            tc::fence_async_smem();
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&bar[4 + k])) : "memory");
        };
        long rk0 = 0, rk1 = 0;  // this row's path, buffers 0 / 1
        bool rl0 = false, rl1 = false;
        double ry0 = 0.0, ry1 = 0.0;
        const uint32_t rbar = tc::smem_u32(&bar[4]), dbar = tc::smem_u32(&bar[0]);
        // register prefetch of a tile's global inputs (issued one iteration ahead)
        struct Pre {
            unsigned short st[kInd];
            double y;
            long k;
            bool live;
        };
        auto fetch = [&](int n) {
            Pre f;
            const long tile = t_first + blockIdx.x + static_cast<long>(n) * gridDim.x;
            const unsigned rw = static_cast<unsigned>(tile * 128) + r;
            f.live = rw >= a.b0 && rw < a.b1;
            f.k = f.live ? rw / static_cast<unsigned>(a.N) : 0;
            f.y = 0.0;
            if (hf == 0) {
#pragma unroll
                for (int c = 0; c < kInd; ++c)
                    f.st[c] = (f.live && c < a.Cc) ? __ldg(a.steps + static_cast<size_t>(c + 1) * a.R + rw) : 0xFFFF;
                if (f.live && (a.mode & 1)) f.y = __ldg(a.y + rw);
            }
            return f;
        };
        // tile n's inputs: default steps -> indicator operand (TMEM)
        auto prep = [&](int n, const Pre& f) {
            const int b = n & 1;
            if (hf == 0) {
                float iv[8];
#pragma unroll
                for (int c = 0; c < kInd; ++c) iv[c] = f.st[c] <= a.step ? 1.0f : 0.0f;
                tc::tmem_st8(tm + b * kEvBuf + lb + 192, iv);
            }
            if (b) rk1 = f.k, rl1 = f.live, ry1 = f.y;
            else rk0 = f.k, rl0 = f.live, ry0 = f.y;
            tc::tmem_wait_st();
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(rbar + 8 * b) : "memory");
        };
        auto layer0 = [&](int n) {  // H1 of tile n -> A[b]
            const int b = n & 1;
            const float4* P = reinterpret_cast<const float4*>(a.Pg + (b ? rk1 : rk0) * kU + cb);
            float4 pg[4];  // the path part, loaded under the D0 wait
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) pg[q4] = __ldg(P + q4);
            tc::mbar_wait_addr(dbar + 8 * b, ph[b]);
            ph[b] ^= 1;
            tc::fence_after_sync();
            float z[16], hi[16], lo[16];
            tc::tmem_ld16(tm + b * kEvBuf + lb + cb, z);
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
                const float4 pv = pg[q4];
                const float pz[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int q = 4 * q4 + u;
                    const float h = act_f<ACT>(z[q] + pz[u]);
                    hi[q] = tc::tf32_rna(h);
                    lo[q] = h - hi[q];
                }
            }
            tc::tmem_st16(tm + b * kEvBuf + lb + 64 + cb, hi);
            tc::tmem_st16(tm + b * kEvBuf + lb + 128 + cb, lo);
            ready(2 + b);
        };
        // H2, f and the requested outputs of tile n; once its accumulator is read, the
        // buffer's next tile n + 2 is prepared (so its D0 runs under this epilogue)
        auto outputs = [&](int n, bool prep_next, const Pre& fn) {
            const int b = n & 1;
            const long tile = t_first + blockIdx.x + static_cast<long>(n) * gridDim.x;
            const long rw = tile * 128 + r;
            const bool live = b ? rl1 : rl0;  // this tile's row state (prep overwrites buffer b's)
            const double yrow = b ? ry1 : ry0;
            wait_done(2 + b);
            float h2[16];
            tc::tmem_ld16(tm + b * kEvBuf + lb + cb, h2);
            if (prep_next) prep(n + 2, fn);
            epi_sync();  // the previous tile's fsh reads are done
            float fp = 0.0f;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                h2[j] = act_f<ACT>(h2[j] + vsh[cb + j]);
                fp = fmaf(h2[j], vsh[kU + cb + j], fp);
            }
            fsh[hf * 128 + r] = fp;
            epi_sync();
            const float f = b2 + ((fsh[r] + fsh[128 + r]) + (fsh[256 + r] + fsh[384 + r]));
            if ((a.mode & 8) && live)
#pragma unroll
                for (int j = 0; j < 16; j += 4)
                    *reinterpret_cast<float4*>(a.H2 + rw * kU + cb + j) = make_float4(h2[j], h2[j + 1], h2[j + 2], h2[j + 3]);
            if (live && hf == 0) {
                const double ph = (f < 0.0f ? 0.0 : static_cast<double>(f)) + mu;
                if (a.mode & 1) {
                    const double res = ph - yrow;
                    loss += res * res;
                }
                if (a.mode & 2) mn = fmin(mn, static_cast<double>(f) + mu);
                if (a.mode & 4) a.pred[rw] = ph;
            }
        };
        epi_sync();  // b1 | w2 staged
        if (nt > 0) prep(0, fetch(0));
        for (int n = 0; n < nt; ++n) {
            Pre f{};
            if (n + 1 < nt) f = fetch(n + 1);  // in flight under layer 0 of n
            layer0(n);
            if (n > 0) outputs(n - 1, n + 1 < nt, f);
            else if (n + 1 < nt) prep(n + 1, f);
        }
        if (nt > 0) outputs(nt - 1, false, Pre{});
    }
    __syncthreads();
    double* red = reinterpret_cast<double*>(fsh);
    loss = warp_sum(loss);
    for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if (lane == 0 && warp < 4) {
        red[warp] = loss;
        red[4 + warp] = mn;
    }
    __syncthreads();
    if (tid == 0) {
        if (a.mode & 1) a.lpart[blockIdx.x] = red[0] + red[1] + red[2] + red[3];
        if (a.mode & 2) a.mpart[blockIdx.x] = fmin(fmin(red[4], red[5]), fmin(red[6], red[7]));
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tm, 512);
}

template <int ACT>
void launch_sgd_act(const SplitArgs& a, long t_first, long n_tiles, int ctas, cudaStream_t s) {
    const size_t smem = sgd_split_smem();
    HCVA_CUDA(cudaFuncSetAttribute(k_sgd_split<ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    pdl_launch(k_sgd_split<ACT>, dim3(ctas), dim3(kSgdThreads + 32), smem, s, a, t_first, n_tiles);
}

template <int ACT>
bool launch_sgd_fused_act(const SplitArgs& a, long t_first, long n_tiles, int ctas, cudaStream_t s) {
    const size_t smem = sgd_split_smem();
    HCVA_CUDA(cudaFuncSetAttribute(k_sgd_split<ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0, dev = 0, sms = 0;
    HCVA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sgd_split<ACT>, kSgdThreads + 32, smem));
    HCVA_CUDA(cudaGetDevice(&dev));
    HCVA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (per_sm < 1 || ctas > per_sm * sms) return false;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(kSgdThreads + 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t err = cudaLaunchKernelEx(&cfg, k_sgd_split<ACT>, a, t_first, n_tiles);
    if (err == cudaErrorCooperativeLaunchTooLarge) {  // not co-resident here: per-step launches instead
        (void)cudaGetLastError();
        return false;
    }
    HCVA_CUDA(err);
    return true;
}

template <int ACT>
void launch_eval_act(const SplitArgs& a, long t_first, long n_tiles, int ctas, cudaStream_t s) {
    const size_t smem = eval_split_smem();
    HCVA_CUDA(cudaFuncSetAttribute(k_eval_split<ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    pdl_launch(k_eval_split<ACT>, dim3(ctas), dim3(kEvThreads + 32), smem, s, a, t_first, n_tiles);
}

}  // namespace

static_assert(sgd_split_smem() <= 227 * 1024, "split SGD kernel exceeds shared memory");
static_assert(2 * kSlots * kU + 2 * kSlots * kQ <= 2 * kPaths * kU, "per-step path parts exceed Psh");
static_assert(2ull * kH >= 128ull * (kU + 1) * 4 + 64 + 4ull * kSlots * kPaths * kQ &&
                  kG >= 128ull * (kInd + kQ + 2) * 4 && kQ % 4 == 0,
              "readout scratch exceeds the operand tiles");
static_assert(eval_split_smem() <= 227 * 1024, "split evaluation kernel exceeds shared memory");

bool split_eligible(int u, int h, int N, int Cc, int q) {
    static const bool on = [] {
        const char* e = std::getenv("HCVA_SPLIT");
        return !(e && e[0] == '0');
    }();
    return on && u == kU && h == 2 && N >= 1 && Cc >= 0 && Cc <= kInd && q >= 1 && q <= kQ;
}

int split_max_ctas(int sm_count) { return 2 * sm_count; }

int launch_sgd_split(const SplitArgs& a, int sm_count, cudaStream_t s) {
    if (a.b1 <= a.b0) throw contract_error("regression tile: empty row range");
    const long t_first = a.b0 / 128, n_tiles = (a.b1 - 1) / 128 - t_first + 1;
    // one CTA per SM, at most sgd_slots tiles each (more CTAs run in later waves)
    const long per = std::min<long>(sgd_slots(a.N), (n_tiles + sm_count - 1) / sm_count);
    const int ctas = static_cast<int>((n_tiles + per - 1) / per);
    switch (a.act) {
        case 0: launch_sgd_act<0>(a, t_first, n_tiles, ctas, s); break;
        case 1: launch_sgd_act<1>(a, t_first, n_tiles, ctas, s); break;
        case 2: launch_sgd_act<2>(a, t_first, n_tiles, ctas, s); break;
        default: launch_sgd_act<3>(a, t_first, n_tiles, ctas, s); break;
    }
    return ctas;
}

bool launch_sgd_split_fused(const SplitArgs& a, int sm_count, cudaStream_t s) {
    if (!a.fuse || a.nsteps < 1 || a.bs < 1 || a.bs % 128 || a.b0 % 128) return false;
    const long t_first = a.b0 / 128, n_tiles = a.bs / 128;  // tiles of each step's batch
    const long per = (n_tiles + sm_count - 1) / sm_count;
    if (per > sgd_slots(a.N)) return false;
    const int ctas = static_cast<int>((n_tiles + per - 1) / per);
    // the fused optimizer gives each thread of a CTA at most one parameter (slices of
    // a multiple of 4 for 16-byte gathers); the gathered rows fill the H1^T tile
    const long pslice = (((a.P + ctas - 1) / ctas + 3) / 4) * 4;
    if (pslice > kSgdThreads + 32 || 4L * ctas * pslice > static_cast<long>(2 * kH)) return false;
    switch (a.act) {
        case 0: return launch_sgd_fused_act<0>(a, t_first, n_tiles, ctas, s);
        case 1: return launch_sgd_fused_act<1>(a, t_first, n_tiles, ctas, s);
        case 2: return launch_sgd_fused_act<2>(a, t_first, n_tiles, ctas, s);
        default: return launch_sgd_fused_act<3>(a, t_first, n_tiles, ctas, s);
    }
}

int launch_eval_split(const SplitArgs& a_in, int sm_count, cudaStream_t s) {
    if (a_in.b1 <= a_in.b0) throw contract_error("regression tile: empty row range");
    SplitArgs a = a_in;
    k_path_proj<<<static_cast<unsigned>((a.M + kPjPaths - 1) / kPjPaths), 256, 0, s>>>(a, a.Pg_out);
    a.Pg = a.Pg_out;
    const long t_first = a.b0 / 128, n_tiles = (a.b1 - 1) / 128 - t_first + 1;
    const int ctas = static_cast<int>(std::min<long>(n_tiles, sm_count));
    switch (a.act) {
        case 0: launch_eval_act<0>(a, t_first, n_tiles, ctas, s); break;
        case 1: launch_eval_act<1>(a, t_first, n_tiles, ctas, s); break;
        case 2: launch_eval_act<2>(a, t_first, n_tiles, ctas, s); break;
        default: launch_eval_act<3>(a, t_first, n_tiles, ctas, s); break;
    }
    return ctas;
}

}  // namespace hcva
