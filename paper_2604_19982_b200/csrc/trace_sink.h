// Host-side forwarding of JoinTrace events (reference JoinTrace, include/trijoin/filter.hpp:56-60).
// Only active when the caller registered callbacks; copies per-op state back after a
// stage and fires events in ascending op order on the calling thread.
#pragma once
#include <vector>

#include "filter.cuh"

namespace tjx {

struct TraceSink {
    void* user = nullptr;
    void (*on_interval)(void*, uint32_t, int16_t, double, double) = nullptr;
    void (*on_vp_pruned)(void*, uint32_t, uint32_t, uint32_t, double, double) = nullptr;

    // Emit on_interval(op, stage, [lb, ub]) for every op with flag[op] != 0.
    void emit_flagged(CandDevStore& cs, const std::vector<uint8_t>& flags, int16_t stage, cudaStream_t st) {
        if (!on_interval || cs.n == 0) return;
        std::vector<double> lb(cs.n), ub(cs.n);
        TJ_CUDA(cudaMemcpyAsync(lb.data(), cs.lb.p, cs.n * 8, cudaMemcpyDeviceToHost, st));
        TJ_CUDA(cudaMemcpyAsync(ub.data(), cs.ub.p, cs.n * 8, cudaMemcpyDeviceToHost, st));
        TJ_CUDA(cudaStreamSynchronize(st));
        for (uint64_t op = 0; op < cs.n; ++op)
            if (flags.empty() || flags[op]) on_interval(user, (uint32_t)op, stage, lb[op], ub[op]);
    }
    void emit_updated(CandDevStore& cs, DevBuf<uint8_t>& updated, int16_t stage, cudaStream_t st) {
        if (!on_interval || cs.n == 0) return;
        std::vector<uint8_t> f(cs.n);
        TJ_CUDA(cudaMemcpyAsync(f.data(), updated.p, cs.n, cudaMemcpyDeviceToHost, st));
        TJ_CUDA(cudaStreamSynchronize(st));
        emit_flagged(cs, f, stage, st);
    }
};

} // namespace tjx
