// common.cuh -- internal structures of libhcva_gpu.so (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>
#include <utility>

#include <nvtx3/nvToolsExt.h>

#include "../../include/hcva_gpu.h"

namespace hcva {

// NVTX range over an engine phase (header-only NVTX3: a no-op unless a tool
// such as Nsight Systems is attached).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Exception types mirroring proj/include/hiercva/errors.hpp:9-25; the C ABI
// converts them to hcva_status codes.
struct config_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct contract_error : std::logic_error { using std::logic_error::logic_error; };
struct numeric_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct cuda_error : std::runtime_error { using std::runtime_error::runtime_error; };

void set_last_error(const std::string& msg);

#define HCVA_CUDA(call)                                                                    \
    do {                                                                                   \
        cudaError_t err__ = (call);                                                        \
        if (err__ != cudaSuccess)                                                          \
            throw ::hcva::cuda_error(std::string(#call) + ": " + cudaGetErrorString(err__)); \
    } while (0)

template <typename F>
hcva_status guarded(F&& f) {
    try {
        f();
        return HCVA_OK;
    } catch (const config_error& e) {
        set_last_error(e.what());
        return HCVA_ERR_CONFIG;
    } catch (const contract_error& e) {
        set_last_error(e.what());
        return HCVA_ERR_CONTRACT;
    } catch (const numeric_error& e) {
        set_last_error(e.what());
        return HCVA_ERR_NUMERIC;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return HCVA_ERR_CUDA;
    }
}

// Host copy of the model with derived quantities.
struct Model {
    int E = 0, Cc = 0, Cn = 0, D = 0;
    std::vector<hcva_vasicek> rates;
    std::vector<hcva_fx> fx;
    std::vector<hcva_cir> credit;
    std::vector<double> corr;  // effective D x D
    std::vector<double> chol;  // lower Cholesky factor
    int n_steps = 0, substeps = 1;
    double dt = 1.0;
};

Model make_model(const hcva_model* m, const hcva_grid* g);  // validates (market.cpp:12-75)
std::vector<double> cholesky_lower(const std::vector<double>& a, int n, const std::string& what);
double zc_price(double r, double tau, const hcva_vasicek& p);
double par_rate(double maturity, double tenor, const hcva_vasicek& p);
bool is_multiple(double x, double step);

// Device-side per-launch constants for the diffusion kernel: per-factor
// coefficient quads staged into shared memory, CSR of the Cholesky factor.
struct FactorCoef {
    double c0, c1, c2, c3;  // Euler coefficients (see prepare_market)
    double v0, v1;          // Cholesky row, when it has <= 2 nonzeros: z = v0 zraw[col0] + v1 zraw[col1]
    int col0, col1;
    int dense;              // row has > 2 nonzeros: use the CSR
    int pad;
};

// Stream the calling C-ABI entry point works on (set by StreamScope); device
// buffers are stream-ordered allocations from the device's memory pool, whose
// release threshold the context raises so repeated runs reuse the memory
// instead of paying cudaMalloc/cudaFree for gigabyte buffers.
cudaStream_t& alloc_stream();

struct StreamScope {
    cudaStream_t prev;
    explicit StreamScope(cudaStream_t s) : prev(alloc_stream()) { alloc_stream() = s; }
    ~StreamScope() { alloc_stream() = prev; }
};

struct DeviceBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaStream_t stream = nullptr;
    void alloc(size_t b) {
        release();
        stream = alloc_stream();
        if (b) HCVA_CUDA(cudaMallocAsync(&p, b, stream));
        bytes = b;
    }
    void release() {
        if (p) cudaFreeAsync(p, stream);
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
    ~DeviceBuf() { release(); }
    DeviceBuf() = default;
    DeviceBuf(const DeviceBuf&) = delete;
    DeviceBuf& operator=(const DeviceBuf&) = delete;
};

}  // namespace hcva

struct hcva_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    uint64_t launches = 0;
    int sm_count = 148;
};

// Simulated set, device resident, SoA with the path index fastest:
//   rates [(i*E + e)*M + k], fx [(i*(E-1) + e-1)*M + k], intens/hazard
//   [(i*Cn + c)*M + k], disc [i*M + k], cube [(i*Cc + c-1)*M + k],
//   default steps [c*R + k*N + l] (uint16, 0xFFFF = survives), R = M*N.
// Lagged rates are not stored: lag(i,e) = rates(i-1,e) for i > 0 and the
// start state's lag (r0 for outer blocks) at i = 0 (market.cpp:186-195).
struct hcva_sim {
    hcva_ctx* ctx = nullptr;
    hcva::Model model;
    int M = 0, n = 0, N = 0, start_step = 0, path_offset = 0;
    int shard_blk = 0, shard_stride = 0;  // interleaved shard map (simulate.cu shard_path)
    int n_groups = 1;  // conditional blocks: states, each with M / n_groups inner paths
    hcva::DeviceBuf rates, fx, intens, hazard, disc, lag0, cube, steps, labels, ties, scratch, profile;
    bool has_cube = false, has_defaults = false;
    int labels_kind = -1;
    // --- execution plan (staged once, reused by every re-run) ---
    // market: per-factor coefficients, Cholesky CSR, initial states, group keys
    hcva::DeviceBuf m_coef, m_row, m_col, m_val, m_init, m_keys;
    int m_nnz = 0, m_T = 0, m_ppg = 1, m_P = 8, m_NT = 128, m_We = 12, m_qcap = 0;
    uint64_t m_local_offset = 0;
    size_t m_smem = 0;
    // MtM: coefficient tables (linear form) or the book (direct form)
    hcva::DeviceBuf c_lnA, c_B, c_dAB, c_Nsuf, c_N, c_NSsuf, c_H, c_book, c_vas;
    bool c_linear = true;
    int c_nswaps = 0;
    // per-phase CUDA events of re-runs: [slot][market, defaults, cube, labels, end]
    std::vector<cudaEvent_t> events;
    ~hcva_sim() {
        for (auto e : events) cudaEventDestroy(e);
    }
};

namespace hcva {

inline unsigned grid1(size_t n, int b) { return static_cast<unsigned>((n + b - 1) / b); }

// Programmatic dependent launch: a kernel launched by pdl_launch may become
// resident while its predecessor drains (the predecessor calls pdl_trigger()),
// runs its prologue, and blocks in pdl_wait() until the predecessor has
// completed and its writes are visible.  No-ops for ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();
template <typename... KArgs, typename... Args>
void pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    HCVA_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// Small host table -> device buffer (stream-ordered, synchronised).
template <typename T>
void stage(DeviceBuf& buf, const std::vector<T>& v) {
    buf.alloc(std::max<size_t>(v.size(), 1) * sizeof(T));
    if (!v.empty()) {
        HCVA_CUDA(cudaMemcpyAsync(buf.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, buf.stream));
        HCVA_CUDA(cudaStreamSynchronize(buf.stream));
    }
}

// Launch helpers shared by the C-ABI translation units (simulate.cu).
void check_launch(hcva_ctx* ctx);
void launch_labels_from(hcva_sim* sim, int kind, int i0, int i1, const uint16_t* steps, int N, double* dev_out);
void probe_block(hcva_sim* sim, uint64_t key, int kind, DeviceBuf& steps, DeviceBuf& labels);
void estimate_qr_device(hcva_ctx* ctx, const double* g /* [n][2] */, size_t n, double* out);  // estimators.cu
void percentile_bands(hcva_ctx* ctx, const double* dev_values, size_t n, double* out /* [5] */);
hcva_sim* new_sim(hcva_ctx* ctx, const hcva_model* model, const hcva_grid* grid);
hcva_sim* new_sim(hcva_ctx* ctx, const Model& model);
void prepare_market(hcva_sim* sim, const std::vector<uint64_t>& group_keys, const std::vector<double>& init_state,
                    int paths_per_group, uint64_t local_offset);
void launch_market(hcva_sim* sim, uint64_t key0);
void prepare_cube(hcva_sim* sim, const hcva_swap* book, int n_swaps);
void launch_cube(hcva_sim* sim);
void copy_out(hcva_ctx* ctx, void* dst, const void* src, size_t bytes);
void launch_labels_all(hcva_sim* sim, int kind);

}  // namespace hcva
