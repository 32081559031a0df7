// TMA (cp.async.bulk.tensor) + mbarrier building blocks for the streaming
// scan kernels, and the host-side tensor-map encoder (driver entry point, so
// the library needs no -lcuda).
//
// The streaming kernels read [rows = B*L, cols = channels] activation planes as
// 2D tensors: one TMA box is PF time steps x LW channels, landing in a shared
// memory stage that the consumer threads read column-wise (thread = channel,
// conflict-free).  A CTA keeps S stages in flight; the full/empty mbarrier
// pair per stage is the producer/consumer handshake.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace lrx {
namespace tma {

// ---------------------------------------------------------------- device
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1, 1000000;\n\t"
        "@!p bra LAB_WAIT;\n\t"
        "}" ::"r"(a),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap* m) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

// 2D tile load: box origin (col c0, row r0) -> dst, completion on bar.
__device__ __forceinline__ void load_2d(void* dst, const CUtensorMap* m, int c0, int r0, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(r0), "r"(smem_u32(bar))
        : "memory");
}

// 3D tile load: box origin (c0, c1, c2) -> dst, completion on bar.  Elements
// outside the tensor are zero-filled (and still count toward complete_tx).
__device__ __forceinline__ void load_3d(void* dst, const CUtensorMap* m, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// 3D tile store smem -> global (bulk group); out-of-bounds parts of the box
// are clipped.  Writers must fence.proxy.async before the issuing barrier.
__device__ __forceinline__ void store_3d(const CUtensorMap* m, const void* src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
                 : "memory");
}
// 1D bulk copy global -> shared (bytes % 16 == 0, 16-byte aligned), completion on bar.
__device__ __forceinline__ void load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// 2D tile store smem -> global (bulk group); out-of-bounds parts clipped.
__device__ __forceinline__ void store_2d(const CUtensorMap* m, const void* src, int c0, int r0) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(c0), "r"(r0), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------- host
// Encode a row-major 2D tensor [rows, cols] of `esize`-byte elements with a
// box of [box_rows, box_cols].  Returns false when the driver entry point is
// unavailable or the encode fails.
bool encode_2d(CUtensorMap* map, const void* base, int esize, uint64_t rows, uint64_t cols, uint32_t box_rows,
               uint32_t box_cols);

// fp32 row-major [rows, cols] with a box of [box_rows, 16 cols = 64 B] and the
// 64-byte swizzle: the K-major SW64 canonical layout of a tcgen05 tf32 operand.
bool encode_2d_f32_sw64(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);

// Encode a row-major 3D tensor [d2, d1, d0] (d0 contiguous) with a box of
// [1, box1, box0]; out-of-bounds box elements read as zero.
bool encode_3d(CUtensorMap* map, const void* base, int esize, uint64_t d2, uint64_t d1, uint64_t d0,
               uint32_t box1, uint32_t box0);

}  // namespace tma
}  // namespace lrx
