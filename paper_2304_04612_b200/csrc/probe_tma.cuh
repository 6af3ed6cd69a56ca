// probe_tma.cuh — TMA read-bandwidth probe (diagnostics, DESIGN.md §6b "short-wide A").
// Streams A (m x k FP32, row stride lda) into shared memory with cp.async.bulk.tensor only — no
// math — using the mainloop's tile order (128-row m-blocks x contiguous k-splits), so the box
// shape (bytes fetched per row per visit) can be varied independently of the GEMM pipeline.
#pragma once
#include <cstdint>
#include <cuda.h>
#include "ptx.cuh"

namespace shg {

constexpr int kProbeStages = 4;
constexpr int kProbeStageBytes = 32768;

// layout 0/1: 2-D map, box {box_k, box_rows}; layout 2: 3-D map {32, k/32, rows}, box
// {32, box_k/32, box_rows}. One box per stage; a 128-row tile takes 128/box_rows boxes per k-step.
__global__ void __launch_bounds__(32, 1)
probe_tma_read_kernel(const __grid_constant__ CUtensorMap map, int layout, int box_k, int box_rows,
                      int m_tiles, int splits, int num_ks, unsigned long long* bytes_out) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* base = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(base + kProbeStages * kProbeStageBytes);
    const uint32_t box_bytes = static_cast<uint32_t>(box_k) * box_rows * 4u;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kProbeStages; ++i) mbar_init(&full[i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    if (threadIdx.x != 0) return;
    const uint64_t pol = policy_evict_first();
    const int groups = 128 / box_rows;
    uint64_t issued = 0;
    for (int tile = blockIdx.x; tile < m_tiles * splits; tile += gridDim.x) {
        const int m_blk = tile / splits, s = tile - (tile / splits) * splits;
        const int ks0 = static_cast<int>((static_cast<int64_t>(s) * num_ks) / splits);
        const int ks1 = static_cast<int>((static_cast<int64_t>(s + 1) * num_ks) / splits);
        for (int ks = ks0; ks < ks1; ++ks) {
            for (int g = 0; g < groups; ++g, ++issued) {
                const uint32_t st = static_cast<uint32_t>(issued % kProbeStages);
                if (issued >= kProbeStages) mbar_wait(&full[st], static_cast<uint32_t>((issued / kProbeStages - 1) & 1));
                mbar_arrive_expect_tx(&full[st], box_bytes);
                void* dst = base + st * kProbeStageBytes;
                const int row = m_blk * 128 + g * box_rows;
                if (layout == 2) tma_load_3d(dst, &map, &full[st], 0, ks * (box_k / 32), row, pol);
                else tma_load_2d(dst, &map, &full[st], ks * box_k, row, pol);
            }
        }
    }
    for (uint64_t j = issued > kProbeStages ? issued - kProbeStages : 0; j < issued; ++j)
        mbar_wait(&full[j % kProbeStages], static_cast<uint32_t>((j / kProbeStages) & 1));
    atomicAdd(bytes_out, static_cast<unsigned long long>(issued) * box_bytes);
}

}  // namespace shg
