// tc.cuh -- thin sm_100a tensor-core layer: tcgen05 MMA (kind::tf32), TMEM,
// mbarriers, shared-memory operand tiles.
//
// Operand tiles use the canonical no-swizzle "core matrix" layout: a logical
// R x C FP32 tile (R % 8 == 0, C % 4 == 0) stores element (r, c) at byte
//   ((c/4) * (R/8) + r/8) * 128 + (r%8) * 16 + (c%4) * 4,
// i.e. 8x4 core matrices of 128 contiguous bytes, consecutive along r, read
// as a K-major operand (rows = M/N, cols = K: SBO = 128, LBO = R/8*128).
// Only K-major operands are used: MN-major reads of these tiles returned
// zeros on sm_100a in our descriptor tests (tools/debug_gemm.py), so
// transposed operands are written transposed instead.
//
// 3xTF32: every FP32 operand is stored as hi = rna_tf32(a) and lo = a - hi;
// D += A_hi B_hi + A_lo B_hi + A_hi B_lo gives ~FP32 products with FP32
// accumulation in TMEM.
#pragma once
#include <cstdint>

namespace hcva {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t core_off(int r, int c, int R) {
    return (static_cast<uint32_t>((c >> 2) * (R >> 3) + (r >> 3)) << 7) + ((r & 7) << 4) + ((c & 3) << 2);
}

// Round to the TF32 grid, ties away from zero (cvt.rna.tf32.f32 without its infinity
// guard: two integer ops; every operand split here is finite -- a non-finite activation
// or gradient is caught by the loss check).
__device__ __forceinline__ float tf32_rna(float a) {
    return __uint_as_float((__float_as_uint(a) + 0x1000u) & 0xFFFFE000u);
}

// Store a into the hi / lo tiles (same layout, `lo_bytes` apart).
__device__ __forceinline__ void put_split(uint8_t* tile, uint32_t lo_bytes, int r, int c, int R, float a) {
    const float hi = tf32_rna(a);
    const uint32_t o = core_off(r, c, R);
    *reinterpret_cast<float*>(tile + o) = hi;
    *reinterpret_cast<float*>(tile + lo_bytes + o) = a - hi;
}

// Four consecutive columns c..c+3 (c % 4 == 0) of row r: one 16-byte store per plane.
__device__ __forceinline__ void put_split4(uint8_t* tile, uint32_t lo_bytes, int r, int c, int R, float4 a) {
    const float4 hi = make_float4(tf32_rna(a.x), tf32_rna(a.y), tf32_rna(a.z), tf32_rna(a.w));
    const uint32_t o = core_off(r, c, R);
    *reinterpret_cast<float4*>(tile + o) = hi;
    *reinterpret_cast<float4*>(tile + lo_bytes + o) = make_float4(a.x - hi.x, a.y - hi.y, a.z - hi.z, a.w - hi.w);
}

__device__ __forceinline__ float get_split(const uint8_t* tile, uint32_t lo_bytes, int r, int c, int R) {
    const uint32_t o = core_off(r, c, R);
    return *reinterpret_cast<const float*>(tile + o) + *reinterpret_cast<const float*>(tile + lo_bytes + o);
}

// UMMA shared-memory descriptor, no swizzle (SmemDescriptor, mma_sm100_desc.hpp).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// Instruction descriptor kind::tf32, D = F32 (InstrDescriptor, mma_sm100_desc.hpp).
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn_major, int b_mn_major) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(a_mn_major) << 15) |
           (static_cast<uint32_t>(b_mn_major) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, int accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accum));
}

// Warp-collective issue: the whole warp evaluates the (warp-uniform)
// descriptors, one elected lane issues.  Keeps descriptor arithmetic in the
// uniform datapath instead of a divergent single-thread branch.
__device__ __forceinline__ uint32_t elect_one() {
    uint32_t e;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(e));
    return e;
}

__device__ __forceinline__ void mma_tf32_if(uint32_t issue, uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                            int accum) {
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "setp.ne.b32 q, %5, 0;\n\t"
        "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accum), "r"(issue));
}

__device__ __forceinline__ void commit_if(uint32_t issue, uint64_t* mbar) {
    asm volatile(
        "{\n\t.reg .pred q;\n\t"
        "setp.ne.b32 q, %1, 0;\n\t"
        "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
            smem_u32(mbar)),
        "r"(issue)
        : "memory");
}

__device__ __forceinline__ void commit(uint64_t* mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(mbar))
                 : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// try_wait's suspend-time hint: a waiting warp is descheduled until the phase
// completes (or this many ns pass) instead of spinning on issue slots.
constexpr uint32_t kSuspendNs = 1000000;

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred done;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1, %2;\n\t"
        "@!done bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(mbar)),
        "r"(parity), "r"(kSuspendNs)
        : "memory");
}

__device__ __forceinline__ void mbar_wait_addr(uint32_t addr, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred done;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1, %2;\n\t"
        "@!done bra WAIT_%=;\n\t}\n" ::"r"(addr),
        "r"(parity), "r"(kSuspendNs)
        : "memory");
}

// Arrive on the barrier announcing `bytes` of asynchronous transfer.
__device__ __forceinline__ void mbar_expect_tx(uint64_t* mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes)
                 : "memory");
}

// Bulk (non-tensor) global -> shared copy completing on `mbar`; 16-byte aligned, bytes % 16 == 0.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(mbar))
        : "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// Warp-wide TMEM allocation of `cols` columns; the base address lands in *dst.
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t base, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols) : "memory");
}

// 16 consecutive FP32 columns of this thread's TMEM lane (warp-collective).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 8 consecutive FP32 columns of this thread's TMEM lane (warp-collective).
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "f"(v[0]),
                 "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}

// Store 16 consecutive FP32 columns of this thread's TMEM lane (warp-collective).
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
        "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Width-generic forms (W = 8 or 16 columns).
template <int W>
__device__ __forceinline__ void tmem_ldw(uint32_t taddr, float* v) {
    if constexpr (W == 8) tmem_ld8(taddr, v);
    else tmem_ld16(taddr, v);
}
template <int W>
__device__ __forceinline__ void tmem_stw(uint32_t taddr, const float* v) {
    if constexpr (W == 8) tmem_st8(taddr, v);
    else tmem_st16(taddr, v);
}


// D[tmem] (+)= A B^T over K (multiple of 8) in 3xTF32, issued by one thread.
// A: M x K tile, B: N x K tile, each given by its hi base address, the byte
// offset of its lo copy, and (for the K walk) whether it is read K-major
// (advance 2 core columns = 2*lbo per K-step) or MN-major (advance one core
// row block = 128 B per K-step).
struct Operand {
    uint32_t hi, lo_off, lbo, sbo;
    int mn_major;
    __device__ __forceinline__ uint64_t desc(int part, int ks) const {
        const uint32_t base = hi + (part ? lo_off : 0u);
        const uint32_t step = mn_major ? 128u * ks : 2u * lbo * ks;
        return sdesc(base + step, lbo, sbo);
    }
};

// Warp-collective gemm3 (call from a whole warp): descriptors from one base
// plus address-field offsets, one elected lane issues every MMA and commits.
__device__ __forceinline__ void gemm3_warp(uint32_t d_tmem, const Operand& A, const Operand& B, int K,
                                           uint32_t idesc, int accumulate, uint64_t* mbar) {
    const uint32_t issue = elect_one();
    const uint64_t a0 = sdesc(A.hi, A.lbo, A.sbo), b0 = sdesc(B.hi, B.lbo, B.sbo);
    const uint64_t al = static_cast<uint64_t>(A.lo_off >> 4), bl = static_cast<uint64_t>(B.lo_off >> 4);
    const uint64_t as = static_cast<uint64_t>(A.mn_major ? 8u : (2u * A.lbo) >> 4);
    const uint64_t bs = static_cast<uint64_t>(B.mn_major ? 8u : (2u * B.lbo) >> 4);
    for (int ks = 0; ks < K / 8; ++ks) {
        const uint64_t da = a0 + as * ks, db = b0 + bs * ks;
        mma_tf32_if(issue, d_tmem, da, db, idesc, (ks > 0 || accumulate) ? 1 : 0);
        mma_tf32_if(issue, d_tmem, da + al, db, idesc, 1);
        mma_tf32_if(issue, d_tmem, da, db + bl, idesc, 1);
    }
    if (mbar) commit_if(issue, mbar);
}

// A operand from tensor memory (TS form): M rows in lanes, K tf32 columns.
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, int accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(accum));
}

// 3xTF32 with A (hi at a_hi, lo at a_lo columns) in tensor memory, B K-major in shared memory.
__device__ __forceinline__ void gemm3_ts(uint32_t d_tmem, uint32_t a_hi, uint32_t a_lo, const Operand& B, int K,
                                         uint32_t idesc, int accumulate) {
    for (int ks = 0; ks < K / 8; ++ks) {
        mma_tf32_ts(d_tmem, a_hi + 8 * ks, B.desc(0, ks), idesc, (ks > 0 || accumulate) ? 1 : 0);
        mma_tf32_ts(d_tmem, a_lo + 8 * ks, B.desc(0, ks), idesc, 1);
        mma_tf32_ts(d_tmem, a_hi + 8 * ks, B.desc(1, ks), idesc, 1);
    }
}

__device__ __forceinline__ void gemm3(uint32_t d_tmem, const Operand& A, const Operand& B, int K, uint32_t idesc,
                                      int accumulate) {
    for (int ks = 0; ks < K / 8; ++ks) {
        mma_tf32(d_tmem, A.desc(0, ks), B.desc(0, ks), idesc, (ks > 0 || accumulate) ? 1 : 0);
        mma_tf32(d_tmem, A.desc(1, ks), B.desc(0, ks), idesc, 1);
        mma_tf32(d_tmem, A.desc(0, ks), B.desc(1, ks), idesc, 1);
    }
}

// ---- 128-byte swizzled tiles (SWIZZLE_128B): rows of 32 FP32 (128 B) in
// 8-row atoms of 1 KB, 16-byte chunk index XOR-ed with the row within the atom.
// Atoms run along the rows first: atom (r/8, c/32) at ((c/32)*(R/8) + r/8)*1024.
// K-major view (rows = M/N, cols = K): SBO = 1024 (next 8 rows), K-step of 8
// FP32 = +32 B inside the atom, +R/8*1024 past each 32 columns.
// MN-major view (rows = K, cols = M/N): SBO = 1024 (next 8 K rows), LBO =
// R/8*1024 (next 32 M/N columns), K-step of 8 = +1024.
__device__ __forceinline__ uint32_t sw_off(int r, int c, int R) {
    const uint32_t atom = static_cast<uint32_t>((c >> 5) * (R >> 3) + (r >> 3)) << 10;
    const uint32_t row = r & 7, chunk = (c & 31) >> 2;
    return atom + (row << 7) + ((chunk ^ row) << 4) + ((c & 3) << 2);
}

__device__ __forceinline__ void put_split_sw(uint8_t* tile, uint32_t lo_bytes, int r, int c, int R, float a) {
    const float hi = tf32_rna(a);
    const uint32_t o = sw_off(r, c, R);
    *reinterpret_cast<float*>(tile + o) = hi;
    *reinterpret_cast<float*>(tile + lo_bytes + o) = a - hi;
}

// Four consecutive columns c..c+3 (c % 4 == 0): one 16-byte chunk per plane.
__device__ __forceinline__ void put_split4_sw(uint8_t* tile, uint32_t lo_bytes, int r, int c, int R, float4 a) {
    const float4 hi = make_float4(tf32_rna(a.x), tf32_rna(a.y), tf32_rna(a.z), tf32_rna(a.w));
    const uint32_t o = sw_off(r, c, R);
    *reinterpret_cast<float4*>(tile + o) = hi;
    *reinterpret_cast<float4*>(tile + lo_bytes + o) = make_float4(a.x - hi.x, a.y - hi.y, a.z - hi.z, a.w - hi.w);
}

__device__ __forceinline__ float get_split_sw(const uint8_t* tile, uint32_t lo_bytes, int r, int c, int R) {
    const uint32_t o = sw_off(r, c, R);
    return *reinterpret_cast<const float*>(tile + o) + *reinterpret_cast<const float*>(tile + lo_bytes + o);
}

__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return sdesc(addr, lbo, sbo) | (2ull << 61);
}

struct OperandSW {
    uint32_t hi, lo_off, R;
    int mn_major;
    __device__ __forceinline__ uint64_t desc(int part, int ks) const {
        const uint32_t base = hi + (part ? lo_off : 0u);
        if (mn_major) return sdesc_sw128(base + 1024u * ks, (R / 8) * 1024u, 1024u);
        const uint32_t col = 8 * ks;  // first K column of this step
        return sdesc_sw128(base + (col >> 5) * (R / 8) * 1024u + (col & 31) * 4u, 16u, 1024u);
    }
};

// Warp-collective gemm3_sw (K-major SW128 operands).
__device__ __forceinline__ void gemm3_sw_warp(uint32_t d_tmem, const OperandSW& A, const OperandSW& B, int K,
                                              uint32_t idesc, int accumulate, uint64_t* mbar) {
    const uint32_t issue = elect_one();
    const uint64_t a0 = A.desc(0, 0), b0 = B.desc(0, 0);
    const uint64_t al = static_cast<uint64_t>(A.lo_off >> 4), bl = static_cast<uint64_t>(B.lo_off >> 4);
    for (int ks = 0; ks < K / 8; ++ks) {
        const uint32_t col = 8 * ks;  // first K column of this step
        const uint64_t da = a0 + ((((col >> 5) * (A.R / 8) * 1024u) + (col & 31) * 4u) >> 4);
        const uint64_t db = b0 + ((((col >> 5) * (B.R / 8) * 1024u) + (col & 31) * 4u) >> 4);
        mma_tf32_if(issue, d_tmem, da, db, idesc, (ks > 0 || accumulate) ? 1 : 0);
        mma_tf32_if(issue, d_tmem, da + al, db, idesc, 1);
        mma_tf32_if(issue, d_tmem, da, db + bl, idesc, 1);
    }
    if (mbar) commit_if(issue, mbar);
}

__device__ __forceinline__ void gemm3_sw(uint32_t d_tmem, const OperandSW& A, const OperandSW& B, int K,
                                         uint32_t idesc, int accumulate) {
    for (int ks = 0; ks < K / 8; ++ks) {
        mma_tf32(d_tmem, A.desc(0, ks), B.desc(0, ks), idesc, (ks > 0 || accumulate) ? 1 : 0);
        mma_tf32(d_tmem, A.desc(1, ks), B.desc(0, ks), idesc, 1);
        mma_tf32(d_tmem, A.desc(0, ks), B.desc(1, ks), idesc, 1);
    }
}

// K-major view of a core tile with R rows; MN-major view of a core tile with R rows.
__device__ __forceinline__ Operand kmajor(const void* hi, uint32_t lo_off, int R) {
    return Operand{smem_u32(hi), lo_off, static_cast<uint32_t>(R / 8) * 128u, 128u, 0};
}
__device__ __forceinline__ Operand mnmajor(const void* hi, uint32_t lo_off, int R) {
    return Operand{smem_u32(hi), lo_off, 128u, static_cast<uint32_t>(R / 8) * 128u, 1};
}

}  // namespace tc
}  // namespace hcva
