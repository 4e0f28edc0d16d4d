// p2p.cu -- fused peer-memory modular all-reduce.
//
// NCCL reduces with +, not + mod q_i (north star), so the baseline cross-rank ciphertext sum
// is an all-gather (R copies land on every rank) followed by ckks_modadd_gathered.  Here
// ONE kernel per rank does the reduction while it moves the data: rank r owns limb rows
// [r S / R, (r + 1) S / R) of the S = count * n_polys * level rows, loads that slice from
// every peer's buffer through CUDA-IPC mappings (NVLink P2P loads), adds mod q_i, and stores
// the sum straight into every peer's output buffer (P2P stores) -- a reduce-scatter and an
// all-gather fused with the modular add.  Per rank, (R-1)/R of the data crosses NVLink
// in each direction, against (R-1) full copies in for the all-gather form.
#include <algorithm>

#include "internal.h"

namespace {

struct PeerPtrs {
    const u64 *in[CKKS_MAX_PEERS];
    u64 *out[CKKS_MAX_PEERS];
};

__global__ void __launch_bounds__(256) k_p2p_modsum(PeerPtrs pp, u32 R, u32 row0, u32 rows, u32 level, u32 cap,
                                                    u32 log_n, const ModC *mod)
{
    const u32 half = 1u << (log_n - 1);  // element pairs per row
    const size_t total = (size_t)rows * half;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const u32 row = row0 + (u32)(e >> (log_n - 1)), k = ((u32)e & (half - 1)) << 1;
        const u32 p = row / level, i = row - p * level;
        const size_t addr = (((size_t)p * cap + i) << log_n) + k;
        const u64 q = mod[i].q;
        u64 s0 = 0, s1 = 0;
        for (u32 r = 0; r < R; ++r) {
            const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(pp.in[r] + addr);
            s0 = csub(s0 + v.x, q);
            s1 = csub(s1 + v.y, q);
        }
        for (u32 r = 0; r < R; ++r) *reinterpret_cast<ulonglong2 *>(pp.out[r] + addr) = make_ulonglong2(s0, s1);
    }
}

}  // namespace

void p2p_slice(u32 rows, u32 R, u32 rank, u32 *row0, u32 *nrows)
{
    const u32 base = rows / R, extra = rows % R;
    *row0 = rank * base + (rank < extra ? rank : extra);
    *nrows = base + (rank < extra ? 1 : 0);
}

void launch_p2p_modsum(const Launch &L, const u64 *const *in, u64 *const *out, u32 R, u32 rank, u32 npolys, u32 level,
                       u32 cap)
{
    PeerPtrs pp{};
    for (u32 r = 0; r < R; ++r) {
        pp.in[r] = in[r];
        pp.out[r] = out[r];
    }
    u32 row0, rows;
    p2p_slice(npolys * level, R, rank, &row0, &rows);
    if (!rows) return;
    const size_t pairs = (size_t)rows << (L.tb->log_n - 1);
    const unsigned blocks = (unsigned)std::min<size_t>((pairs + 255) / 256, (size_t)L.n_sm * 16);
    const double n = (double)rows * (1u << L.tb->log_n);
    KLAUNCH(L, "p2p_modsum", (Work{0, 0, 8.0 * n * 2 * R}),
            (k_p2p_modsum<<<blocks, 256, 0, L.st>>>(pp, R, row0, rows, level, cap, L.tb->log_n, L.tb->mod)));
}
