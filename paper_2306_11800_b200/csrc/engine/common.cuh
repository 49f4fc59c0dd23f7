// Shared definitions for the dqtg engine (B200 / sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "dqtg.h"

namespace dqtg {

// Internal exception carrying a dqtg_status; converted at the C-ABI boundary.
struct Fail : std::runtime_error {
    dqtg_status code;
    Fail(dqtg_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define DQTG_CUDA(call)                                                                     \
    do {                                                                                    \
        cudaError_t err_ = (call);                                                          \
        if (err_ != cudaSuccess)                                                            \
            throw ::dqtg::Fail(DQTG_CUDA, std::string(#call) + ": " + cudaGetErrorString(err_)); \
    } while (0)

#define DQTG_REQUIRE(cond, code, msg)                     \
    do {                                                  \
        if (!(cond)) throw ::dqtg::Fail((code), (msg));   \
    } while (0)

constexpr int kLayerTypes = 7;
constexpr int kEmbedding = 4;

// Padded flat layout: every tensor starts on a 64-element boundary so tiles are
// 128-byte aligned for fp32 and u16 streams.
constexpr uint64_t kAlign = 64;

// Device-side error word bits (checked by the host after each pipeline).
enum DevErr : uint32_t {
    kErrEmptySketch = 1u << 0,
    kErrCorruptIndex = 1u << 1,
    kErrHuffmanDepth = 1u << 2,
    kErrNonFinite = 1u << 3,
    kErrKmeansWeights = 1u << 4,
    kErrCorruptBitstream = 1u << 5,
};

inline uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }
inline uint64_t ceil_div(uint64_t x, uint64_t a) { return (x + a - 1) / a; }

// ---- device helpers ------------------------------------------------------
__device__ __forceinline__ uint16_t bf16_rne(float v) {  // quantize.cpp:337-342
    uint32_t bits = __float_as_uint(v);
    bits += 0x7fffu + ((bits >> 16) & 1u);
    return (uint16_t)(bits >> 16);
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ uint32_t warp_xor(uint32_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v ^= __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Exclusive block scan of one value per thread (blockDim multiple of 32, <= 1024).
template <typename T>
__device__ T block_exclusive_scan(T v, T* smem /* >= 33 */, T* total = nullptr) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) smem[wid] = x;
    __syncthreads();
    if (wid == 0) {
        T s = lane < nw ? smem[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) smem[lane] = s;  // inclusive per-warp prefix
        if (lane == nw - 1) smem[32] = s;
    }
    __syncthreads();
    T base = wid ? smem[wid - 1] : T(0);
    T out = base + x - v;
    if (total) *total = smem[32];
    __syncthreads();
    return out;
}

// Bulk L2 prefetch (TMA engine, one instruction per region): the next tile's
// inputs are in L2 by the time the CTA's loads reach them.  addr 16-B aligned,
// bytes a multiple of 16.
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// ---- bulk copies global -> shared (TMA engine) with mbarrier completion -----------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
// the calling thread arrives and arms the barrier with the bytes the copies will deliver
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* m, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes)
                 : "memory");
}
// dst / src 16-B aligned, bytes a multiple of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(m))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(m)),
        "r"(parity)
        : "memory");
}
// generic-proxy reads of a buffer before the async proxy (bulk copies) rewrites it
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Dynamic tile scheduling for persistent CTAs: each grab takes `grab` consecutive
// tiles from a global counter (zeroed before the launch), so a kernel sharing the
// GPU with another stream's work load-balances instead of waiting on late CTAs.
// Block-uniform; call from all threads.
__device__ __forceinline__ int grab_tiles(unsigned int* ctr, int grab, int* s_base) {
    __syncthreads();
    if (threadIdx.x == 0) *s_base = (int)atomicAdd(ctr, (unsigned int)grab);
    __syncthreads();
    return *s_base;
}

}  // namespace dqtg
