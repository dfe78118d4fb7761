// common.cuh -- small device helpers shared by the bsrprune kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace bsrp {

constexpr int kWarp = 32;

// Element traits: fp32 or bf16 stored as raw 16-bit patterns.
template <int ES> struct Elem;
template <> struct Elem<4> {
    __device__ __forceinline__ static float to_f32(uint32_t bits) { return __uint_as_float(bits); }
};
template <> struct Elem<2> {
    __device__ __forceinline__ static float to_f32(uint32_t bits16) { return __uint_as_float(bits16 << 16); }
};

// Raw vector of VB bytes (4, 8 or 16); moved as integers so that -0.0,
// denormals and NaN payloads are copied bit-exactly.
template <int VB> struct Vec;
template <> struct Vec<16> { using T = uint4; };
template <> struct Vec<8> { using T = uint2; };
template <> struct Vec<4> { using T = uint32_t; };

template <typename V>
__device__ __forceinline__ V ld_stream(const V *p) {  // read-once data: skip L1
    return __ldcs(p);
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t *p) { return __ldcs(reinterpret_cast<const unsigned int *>(p)); }

// 32-bit words of a vector.
__device__ __forceinline__ uint32_t word(const uint4 &v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}
__device__ __forceinline__ uint32_t word(const uint2 &v, int i) { return i == 0 ? v.x : v.y; }
__device__ __forceinline__ uint32_t word(const uint32_t &v, int) { return v; }

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid-wide barrier for a cooperatively launched (co-resident) grid.  The
// counter is monotonic within one launch and zeroed before the launch;
// barrier number `i` (0-based) completes when (i+1)*gridDim.x arrivals exist.
// Release/acquire (the CUTLASS generic-barrier pattern): bar.sync orders the
// CTA's writes before thread 0's red.release, thread 0's ld.acquire orders the
// other CTAs' writes before the closing bar.sync -- no full fences.
__device__ __forceinline__ void grid_barrier(uint32_t *counter, uint32_t index) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(counter), "r"(1u) : "memory");
        const uint32_t target = (index + 1u) * gridDim.x;
        uint32_t spins = 0;
        while (ld_acquire_gpu(counter) < target) {
            if (++spins > (1u << 26)) __trap();  // workspace not zero-filled / corrupted: fail, do not hang
        }
    }
    __syncthreads();
}

// Programmatic dependent launch (PDL): a kernel launched with
// launch_pdl() may start while its stream predecessor drains; it must call
// pdl_wait() before its first global-memory access (the wait returns once the
// predecessor grid has completed and its writes are visible).  pdl_trigger()
// lets the successor's CTAs be scheduled before this grid exits.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

}  // namespace bsrp
