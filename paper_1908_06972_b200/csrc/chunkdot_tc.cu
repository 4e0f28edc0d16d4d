// chunkdot_tc.cu -- PrivFT's v.H chunk-dot on the tensor cores (P:213
// "a_j = sum_k HMULPLAIN(ct_k, P^H_{j,k})").
//
// At every coefficient position p = (limb i, index n) of the NTT domain the chunk-dot is a
// dense integer matrix product
//      C_p[(b, poly)][j] = sum_k A_p[(b, poly)][k] * H_p[k][j]   (mod q_i)
// with A_p = the query bags (M = 2B rows), H_p = the packed model (J = n columns), K chunks.
// Residues are split into U = ceil(bits(q_i) / 8) byte planes, x = sum_u 2^{8u} x_u, so
//      A H = sum_{s=0}^{2U-2} 2^{8s} sum_{u+v=s} A_u H_v
// and every A_u H_v is an exact u8 x u8 -> s32 tensor-core product (mma.sync m16n8k32; the
// s32 sums stay below U * K * 255^2 < 2^31 for K <= 4096).  The plane classes are folded as
// sum_s c_s [2^{8s} mod q_i] in a 128-bit accumulator (< (2U-1) 2^31 q < 2^97, any K) and
// reduced mod q_i once: bit-identical to the modular multiply-accumulate it replaces.  (The
// plain sum_s c_s 2^{8s} = A H itself reaches K q^2 and wraps 2^128 for K >= 256 at 60 bits.)
//
// Operands: H is re-laid once per model (ckks_privft_model_*) into mma B-fragment order
//   Hf[limb i][plane v][n][j-tile][k-step][lane][2 words]  (256 B per fragment, coalesced);
// A is split per position into shared memory (row pitch padded for conflict-free loads).
// One CTA per position, 8 warps over 16 x (8 NJ) output tiles; per k-step a warp loads the U
// A fragments (ldmatrix) and U NJ B fragments once and issues all U^2 NJ products into the
// 2U-1 plane-class accumulators held in registers.
#include <algorithm>

#include "internal.h"

namespace {

constexpr int TC_THREADS = 256;

__device__ __forceinline__ void mma_u8(int c[4], const unsigned a[4], unsigned b0, unsigned b1)
{
    asm(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// byte u of four consecutive residues, packed little-endian (lowest k in the lowest byte)
__device__ __forceinline__ unsigned pack_plane(const u64 x[4], int u)
{
    const int sh = 8 * u;
    return (unsigned)((x[0] >> sh) & 0xff) | (unsigned)((x[1] >> sh) & 0xff) << 8 |
           (unsigned)((x[2] >> sh) & 0xff) << 16 | (unsigned)((x[3] >> sh) & 0xff) << 24;
}

// ---- H re-layout: one warp = 4 consecutive positions x 8 consecutive fragment words ---------
// word w (0..63) of fragment (jt, ks): lane = w / 2, reg = w % 2;
// B[k][col]: col = jt*8 + lane/4, k = ks*32 + reg*16 + (lane%4)*4 + e (e = byte 0..3)
__global__ void __launch_bounds__(256) k_chunkdot_prep_h(const u64 *H, u32 h_cap, u32 *Hf, u32 i, u32 U, u32 J, u32 K,
                                                        u32 JT, u32 KS, u32 log_n, size_t total)
{
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= total) return;
    const u32 lane32 = (u32)(t & 31);
    const size_t wg = t >> 5;  // (frag, wgrp, n / 4)
    const u32 n = (u32)((wg % ((1u << log_n) / 4)) * 4 + lane32 / 8);
    const size_t fw = wg / ((1u << log_n) / 4);  // (jt, ks, wgrp)
    const u32 wgrp = (u32)(fw % 8), frag = (u32)(fw / 8);
    const u32 ks = frag % KS, jt = frag / KS;
    const u32 w = wgrp * 8 + (lane32 & 7), lane = w / 2, reg = w % 2;
    const u32 col = jt * 8 + lane / 4;
    const u32 k0 = ks * 32 + reg * 16 + (lane % 4) * 4;
    u64 x[4] = {0, 0, 0, 0};
    if (col < J)
        for (int e = 0; e < 4; ++e)
            if (k0 + e < K) x[e] = H[((((size_t)col * K + k0 + e) * h_cap + i) << log_n) + n];
    const size_t nn = (size_t)1 << log_n;
    for (u32 v = 0; v < U; ++v)
        Hf[((((size_t)v * nn + n) * JT + jt) * KS + ks) * 64 + w] = pack_plane(x, (int)v);
}

struct TcArgs {
    const u64 *ct;  // [M/2 * K][2][ct_cap][N]
    const u32 *Hf;  // this limb's fragments
    u64 *out;       // [B * J][2][out_cap][N]
    u32 ct_cap, out_cap, B, J, K, JT, KS, i, log_n;
};

template <int U>
__global__ void __launch_bounds__(TC_THREADS, 2) k_chunkdot_tc(TcArgs a, const ModC *mods)
{
    extern __shared__ u32 As[];  // [U][Mp][pitch] words, pitch = KS*8 + 4
    const u32 n = blockIdx.x;
    const u32 M = 2 * a.B, MT = (M + 15) / 16, Mp = MT * 16;
    const u32 pitch = a.KS * 8 + 4, kgs = a.KS * 8;
    const size_t nn = (size_t)1 << a.log_n;
    // phase 1: this position's A, split into byte planes
    for (u32 idx = threadIdx.x; idx < Mp * kgs; idx += TC_THREADS) {
        const u32 r = idx / kgs, kg = idx % kgs, b = r >> 1, poly = r & 1;
        u64 x[4] = {0, 0, 0, 0};
        if (r < M)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const u32 k = kg * 4 + e;
                if (k < a.K) x[e] = __ldg(a.ct + ((((size_t)(b * a.K + k) * 2 + poly) * a.ct_cap + a.i) << a.log_n) + n);
            }
#pragma unroll
        for (int u = 0; u < U; ++u) As[((size_t)u * Mp + r) * pitch + kg] = pack_plane(x, u);
    }
    __syncthreads();
    const ModC m = load_mod(mods, a.i);
    const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
    constexpr int NJ = U <= 5 ? 2 : 1;  // j-tiles per warp tile (register budget of the class sums)
    constexpr int NC = 2 * U - 1;       // plane classes s = u + v
    const u32 JTW = (a.JT + NJ - 1) / NJ;
    u64 pw[NC];  // 2^{8s} mod q_i
    pw[0] = 1;
#pragma unroll
    for (int s = 1; s < NC; ++s) pw[s] = mulmod(pw[s - 1], 256, m);
    const u32 *hf_n = a.Hf + (size_t)n * a.JT * a.KS * 64 + lane * 2;
    const size_t plane_stride = nn * a.JT * a.KS * 64;
    const u32 pitch_b = pitch * 4;
    // ldmatrix.x4 row address of this lane: rows (lane & 15), k-bytes +16 for lanes 16..31
    const u32 sm_base = (u32)__cvta_generic_to_shared(As) + (lane & 15) * pitch_b + (lane >> 4) * 16;
    for (u32 tile = warp; tile < MT * JTW; tile += TC_THREADS / 32) {
        const u32 mt = tile % MT, jw = tile / MT;
        u32 jt[NJ];
#pragma unroll
        for (int y = 0; y < NJ; ++y) jt[y] = (jw * NJ + y < a.JT) ? jw * NJ + y : a.JT - 1;
        int c[NC][NJ][4];
#pragma unroll
        for (int s = 0; s < NC; ++s)
#pragma unroll
            for (int y = 0; y < NJ; ++y)
#pragma unroll
                for (int e = 0; e < 4; ++e) c[s][y][e] = 0;
        const u32 a_tile = sm_base + mt * 16 * pitch_b;
        for (u32 ks = 0; ks < a.KS; ++ks) {
            unsigned af[U][4];
            uint2 bf[U][NJ];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const u32 addr = a_tile + (u32)u * Mp * pitch_b + ks * 32;
                asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                             : "=r"(af[u][0]), "=r"(af[u][1]), "=r"(af[u][2]), "=r"(af[u][3])
                             : "r"(addr));
            }
#pragma unroll
            for (int v = 0; v < U; ++v)
#pragma unroll
                for (int y = 0; y < NJ; ++y)
                    bf[v][y] = __ldg(reinterpret_cast<const uint2 *>(hf_n + v * plane_stride +
                                                                      ((size_t)jt[y] * a.KS + ks) * 64));
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int v = 0; v < U; ++v)
#pragma unroll
                    for (int y = 0; y < NJ; ++y) mma_u8(c[u + v][y], af[u], bf[v][y].x, bf[v][y].y);
        }
        // fold the plane classes: sum_s c_s [2^{8s} mod q] (< 2^97 for any K), reduce once
#pragma unroll
        for (int y = 0; y < NJ; ++y)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                Acc128 acc;
#pragma unroll
                for (int s = 0; s < NC; ++s) acc.mac((u64)(unsigned)c[s][y][e], pw[s]);
                const u32 row = mt * 16 + g + ((e & 2) ? 8 : 0);
                const u32 col = (jw * NJ + y) * 8 + tq * 2 + (e & 1);
                if (row < M && col < a.J) {
                    const u32 b = row >> 1, poly = row & 1;
                    a.out[((((size_t)b * a.J + col) * 2 + poly) * a.out_cap + a.i) << a.log_n | n] =
                        acc.reduce(m);
                }
            }
    }
}

template <int U>
void tc_launch(const Launch &L, const TcArgs &a, double macs)
{
    const u32 MT = (2 * a.B + 15) / 16;
    const size_t smem = (size_t)U * MT * 16 * (a.KS * 8 + 4) * sizeof(u32);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_chunkdot_tc<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    const double pos = (double)(1u << a.log_n);
    // bytes per position: A (2B x K words), H fragments (JT*8 x KS*32 x U bytes), C (2B x J words)
    const double bytes = pos * (16.0 * a.B * a.K + (double)a.JT * 8 * a.KS * 32 * U + 16.0 * a.B * a.J);
    KLAUNCH(L, "chunkdot_tc", (Work{0, macs, bytes}),
            (k_chunkdot_tc<U><<<1u << a.log_n, TC_THREADS, smem, L.st>>>(a, L.tb->mod)));
}

}  // namespace

u32 chunkdot_tc_planes(u64 q)
{
    u32 bits = 0;
    while (bits < 64 && (q >> bits)) ++bits;
    return (bits + 7) / 8;
}

size_t chunkdot_tc_words(const u64 *hprimes, u32 l, u32 J, u32 K, u32 log_n)
{
    const size_t JT = (J + 7) / 8, KS = (K + 31) / 32;
    size_t w = 0;
    for (u32 i = 0; i < l; ++i) w += (size_t)chunkdot_tc_planes(hprimes[i]) * ((size_t)1 << log_n) * JT * KS * 64;
    return w;
}

bool chunkdot_tc_supported(const u64 *hprimes, u32 l, u32 B, u32 K)
{
    if (K < 1 || K > 4096 || B < 1) return false;
    const u32 MT = (2 * B + 15) / 16, KS = (K + 31) / 32;
    for (u32 i = 0; i < l; ++i) {
        const u32 U = chunkdot_tc_planes(hprimes[i]);
        if (U < 4 || U > 8) return false;
        if ((size_t)U * MT * 16 * (KS * 8 + 4) * 4 > 200 * 1024) return false;
    }
    return true;
}

void launch_chunkdot_prep_h(const Launch &L, const u64 *H, u32 h_cap, u32 *Hf, u32 l, u32 J, u32 K)
{
    const u32 log_n = L.tb->log_n, JT = (J + 7) / 8, KS = (K + 31) / 32;
    size_t off = 0;
    for (u32 i = 0; i < l; ++i) {
        const u32 U = chunkdot_tc_planes(L.hprimes[i]);
        const size_t total = (size_t)JT * KS * 8 * ((1u << log_n) / 4) * 32;
        KLAUNCH(L, "chunkdot_prep_h", (Work{0, 0, 8.0 * J * K * (1u << log_n)}),
                (k_chunkdot_prep_h<<<(unsigned)((total + 255) / 256), 256, 0, L.st>>>(H, h_cap, Hf + off, i, U, J, K, JT,
                                                                                     KS, log_n, total)));
        off += (size_t)U * ((size_t)1 << log_n) * JT * KS * 64;
    }
}

void launch_chunkdot_tc(const Launch &L, const u64 *ct, u32 ct_cap, const u32 *Hf, u64 *out, u32 out_cap, u32 B,
                        u32 J, u32 K, u32 l)
{
    const u32 log_n = L.tb->log_n, JT = (J + 7) / 8, KS = (K + 31) / 32;
    size_t off = 0;
    for (u32 i = 0; i < l; ++i) {
        const u32 U = chunkdot_tc_planes(L.hprimes[i]);
        const TcArgs a{ct, Hf + off, out, ct_cap, out_cap, B, J, K, JT, KS, i, log_n};
        const double macs = 2.0 * B * J * K * (double)(1u << log_n);
        switch (U) {
        case 4: tc_launch<4>(L, a, macs); break;
        case 5: tc_launch<5>(L, a, macs); break;
        case 6: tc_launch<6>(L, a, macs); break;
        case 7: tc_launch<7>(L, a, macs); break;
        default: tc_launch<8>(L, a, macs); break;
        }
        off += (size_t)U * ((size_t)1 << log_n) * JT * KS * 64;
    }
}
