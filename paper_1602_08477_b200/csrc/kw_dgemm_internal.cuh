// kw_dgemm_internal.cuh — the DGEMM translation units' shared interface: the kernel parameter
// block and the entry points the host-operand schedules (kw_dgemm_e2e.cu) and the row-sharded
// driver (kw_comm.cu) call; kernels and their configurations stay private to kw_dgemm.cu.
#pragma once

#include "kw_common.cuh"

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace kw::gemm {

struct GemmParams {
    int m, n, k;
    double alpha, beta;
    const double* a;
    long long lda;
    const double* b;
    long long ldb;
    double* c;
    long long ldc;
    int tiles_m, tiles_n;
    // Streamed mode (host-resident operands, dgemm_streamed): the copy stream uploads A in row
    // panels, B in column panels and C in blocks, and publishes each with a stream write of
    // ready[] = 1: [pass 0: npr A | npc B] ... [pass P-1: npr A | npc B][npr*npc C blocks],
    // followed by the done[npr*npc] counters and one abort word (a ready-flag wait that timed
    // out writes KW_FAIL_READY_TIMEOUT there). The persistent kernel walks tile_list
    // (tile_list[0] = {entry count, P}, then entries {tile row, tile col, first k-tile, end
    // k-tile | pass << 27}; tile row < 0 = padding) in availability order and waits for a tile's
    // panels of the entry's pass before loading them. A tile runs as P entries over consecutive
    // k-ranges (k-split): all but the last park their accumulators in `partial`, all but the
    // first reload them — same thread, same DMMA order, no bit changes. Every consumer warp of a
    // tile's last entry bumps done[block] after storing its part of the block, which releases
    // the block's download. nullptr = ordinary launch (operands resident).
    // (The struct size is part of the tuned kernels' codegen: measured, a larger parameter block
    // costs the resident DGEMM 1.3 % — keep new streamed fields out of it.)
    const int4* tile_list;
    uint32_t* ready;
    double* partial;
    int panel_rows, panel_cols, npr, npc;
};


GemmParams make_params(size_t m, size_t n, size_t k, double alpha, const double* A, size_t lda, const double* B,
                       size_t ldb, double beta, double* C, size_t ldc);
size_t round2(size_t v); // leading dimension rounded up to a 16-byte multiple of doubles
// One launch of the tiled DGEMM (the CTA tile chosen per problem; tile 64 forces the 64 x 64 one).
kw_status launch_tiled(cudaStream_t s, int tile, const GemmParams& p);
kw_status launch_tiled_dp(cudaStream_t s, int tile, const GemmParams& p); // data-parallel configs only
bool tma_eligible(const GemmParams& p);

// Streamed mode: the configuration the persistent launch uses, its tile and consumer warps
// (done[] counts one arrival per consumer warp per tile), and the launch itself.
struct StreamedShape {
    int bm, bn;
    uint32_t consumers;
};
int streamed_config(int tile, const GemmParams& p);
StreamedShape streamed_shape(int cfg);
// The persistent grid launch_streamed uses for this problem (entry e of the tile list runs on
// CTA e mod grid: a k-split pads its first pass to a multiple of it so both passes of a tile
// run on the same CTA).
int streamed_grid(int cfg, const GemmParams& p);
kw_status launch_streamed(cudaStream_t s, int cfg, const GemmParams& p);

// Host-operand schedules (kw_dgemm_e2e.cu): row panels, and the streamed schedule (returns
// KW_OK with *used = false, nothing enqueued, when it does not apply).
kw_status dgemm_staged(kw::Queue* q, int tile, size_t m, size_t n, size_t k, double alpha, const double* A,
                       size_t lda, const double* B, size_t ldb, double beta, double* C, size_t ldc, bool a_dev,
                       bool b_dev, bool c_dev);
kw_status dgemm_streamed(kw::Queue* q, int tile, size_t m, size_t n, size_t k, double alpha, const double* A,
                         size_t lda, const double* B, size_t ldb, double beta, double* C, size_t ldc, bool* used);

} // namespace kw::gemm
