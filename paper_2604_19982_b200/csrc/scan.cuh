// Prefix scans and stable stream compaction on the device (the reference's parcore scans and
// compact_par, proj/include/trijoin/parcore.hpp:59-146, used by voxel_pair_compact / the
// active-list erase_if, src/filter.cpp:265-315, src/refine.cpp:299-301): three passes over
// tiles of kScanTile items — per-tile totals, one block scanning the tile totals, then each
// tile rescanned and written with its offset. Stable (items keep their order), exact
// (64-bit integer sums), and no temporary beyond one u64 per tile.
#pragma once
#include <cstdint>

#include "tj_internal.cuh"

namespace tjx {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8; // consecutive items per thread
constexpr int kScanTile = kScanThreads * kScanItems;

// Exclusive block-wide scan of one u64 per thread (kScanThreads threads); *total = block sum.
__device__ inline uint64_t block_excl_scan(uint64_t v, uint64_t* warp_sums, uint64_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint64_t w = lane < kScanThreads / 32 ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t x = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += x;
        }
        if (lane < kScanThreads / 32) warp_sums[lane] = w; // inclusive warp prefixes
    }
    __syncthreads();
    const uint64_t before = warp ? warp_sums[warp - 1] : 0;
    *total = warp_sums[kScanThreads / 32 - 1];
    __syncthreads(); // warp_sums may be reused by the caller's next scan
    return before + incl - v;
}

// Pass 1: sums[t] = sum of tile t of in (items converted to u64 by Get).
template <class Get>
__global__ void __launch_bounds__(kScanThreads) k_tile_sums(Get get, uint64_t n, uint64_t* __restrict__ sums) {
    __shared__ uint64_t ws[32];
    const uint64_t t0 = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
    uint64_t v = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
        if (t0 + k < n) v += get(t0 + k);
    uint64_t total;
    block_excl_scan(v, ws, &total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// Pass 2 (one block): sums[0, nt) -> exclusive offsets in place; sums[nt] = grand total.
static __global__ void __launch_bounds__(kScanThreads) k_scan_tile_sums(uint64_t* __restrict__ sums, uint64_t nt) {
    __shared__ uint64_t ws[32];
    uint64_t carry = 0;
    for (uint64_t b = 0; b < nt; b += kScanThreads) {
        const uint64_t i = b + threadIdx.x;
        const uint64_t v = i < nt ? sums[i] : 0;
        uint64_t total;
        const uint64_t ex = block_excl_scan(v, ws, &total);
        if (i < nt) sums[i] = carry + ex;
        carry += total;
    }
    if (threadIdx.x == 0) sums[nt] = carry;
}

// Pass 3 (scan): out[i + 1] = inclusive prefix of item i (out[0] written by the caller).
template <class Get>
__global__ void __launch_bounds__(kScanThreads) k_tile_scan(Get get, uint64_t n, const uint64_t* __restrict__ offs,
                                                            uint64_t* __restrict__ out) {
    __shared__ uint64_t ws[32];
    const uint64_t t0 = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
    uint64_t v[kScanItems], sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = t0 + k < n ? get(t0 + k) : 0;
        sum += v[k];
    }
    uint64_t total;
    uint64_t run = offs[blockIdx.x] + block_excl_scan(sum, ws, &total);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        run += v[k];
        if (t0 + k < n) out[t0 + k + 1] = run;
    }
}

// Pass 3 (select): items i with keep(i) written in order to out[offs[tile] + ...].
template <class Keep, class Emit>
__global__ void __launch_bounds__(kScanThreads) k_tile_select(Keep keep, Emit emit, uint64_t n,
                                                              const uint64_t* __restrict__ offs) {
    __shared__ uint64_t ws[32];
    const uint64_t t0 = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
    uint32_t bits = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
        if (t0 + k < n && keep(t0 + k)) bits |= 1u << k;
    uint64_t total;
    uint64_t pos = offs[blockIdx.x] + block_excl_scan((uint64_t)__popc(bits), ws, &total);
    while (bits) {
        const int k = __ffs(bits) - 1;
        bits &= bits - 1;
        emit(t0 + k, pos++);
    }
}

// Predicate as a 0/1 count (pass 1 of a select).
template <class Keep>
struct KeepCount {
    Keep keep;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return keep(i) ? 1u : 0u; }
};

// Inclusive scan of n items (get(i) -> u64) into out[1, n]; out[0] = 0. Returns the total
// (stream-synchronous). tiles: grow-only scratch (one u64 per tile + 1).
template <class Get>
inline uint64_t device_scan(Get get, uint64_t n, uint64_t* out, DevBuf<uint64_t>& tiles, int num_sms, cudaStream_t st) {
    (void)num_sms;
    TJ_CUDA(cudaMemsetAsync(out, 0, sizeof(uint64_t), st));
    if (n == 0) return 0;
    const uint64_t nt = (n + kScanTile - 1) / kScanTile;
    tiles.reserve(nt + 1);
    count_launch();
    k_tile_sums<<<(unsigned)nt, kScanThreads, 0, st>>>(get, n, tiles.p);
    count_launch();
    k_scan_tile_sums<<<1, kScanThreads, 0, st>>>(tiles.p, nt);
    count_launch();
    k_tile_scan<<<(unsigned)nt, kScanThreads, 0, st>>>(get, n, tiles.p, out);
    TJ_CUDA(cudaGetLastError());
    uint64_t total = 0;
    TJ_CUDA(cudaMemcpyAsync(&total, out + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    stream_sync(st);
    return total;
}

// Stable selection: emit(i, k) for the k-th item i (ascending) with keep(i). Returns the count
// (stream-synchronous).
template <class Keep, class Emit>
inline uint64_t device_select(Keep keep, Emit emit, uint64_t n, DevBuf<uint64_t>& tiles, cudaStream_t st) {
    if (n == 0) return 0;
    const uint64_t nt = (n + kScanTile - 1) / kScanTile;
    tiles.reserve(nt + 1);
    count_launch();
    k_tile_sums<<<(unsigned)nt, kScanThreads, 0, st>>>(KeepCount<Keep>{keep}, n, tiles.p);
    count_launch();
    k_scan_tile_sums<<<1, kScanThreads, 0, st>>>(tiles.p, nt);
    count_launch();
    k_tile_select<<<(unsigned)nt, kScanThreads, 0, st>>>(keep, emit, n, tiles.p);
    TJ_CUDA(cudaGetLastError());
    uint64_t total = 0;
    TJ_CUDA(cudaMemcpyAsync(&total, tiles.p + nt, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    stream_sync(st);
    return total;
}

} // namespace tjx
