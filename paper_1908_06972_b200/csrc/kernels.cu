// kernels.cu -- the sm_100a kernels of libckks and their launchers.
//
//   NTT family:  k_fwd_cols / k_fwd_rows_store, k_inv_rows / k_inv_cols
//   rescale + ModDown epilogue (a3, a4):  k_fwd_cols<TaskBcast> + k_fwd_rows_submul
//   key switch ModUp + inner product (a4): k_fwd_cols<TaskModUp> + k_ks_mac
//   limb-wise modular arithmetic (a2): k_elem<...>
//
// Geometry and arithmetic conventions are documented in ntt.cuh / modarith.cuh.
#include <type_traits>

#include "internal.h"

#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

struct Prof {
    bool on = false;
    struct Rec {
        const char *name;
        cudaEvent_t a, b;
        Work w;
    };
    std::vector<Rec> pending;
    std::vector<cudaEvent_t> pool;
    std::map<std::string, ProfTotal> acc;
    const char *cur = nullptr;
    Work cur_w{};
    cudaEvent_t cur_a = nullptr;
    cudaEvent_t get()
    {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
};

void prof_begin(Prof *p, cudaStream_t st, const char *name, Work w)
{
    if (!p || !p->on) return;
    p->cur = name;
    p->cur_w = w;
    p->cur_a = p->get();
    cudaEventRecord(p->cur_a, st);
}

void prof_end(Prof *p, cudaStream_t st)
{
    if (!p || !p->on || !p->cur) return;
    cudaEvent_t b = p->get();
    cudaEventRecord(b, st);
    p->pending.push_back(Prof::Rec{p->cur, p->cur_a, b, p->cur_w});
    p->cur = nullptr;
}

Prof *prof_create() { return new Prof(); }
void prof_destroy(Prof *p)
{
    if (!p) return;
    for (auto &r : p->pending) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : p->pool) cudaEventDestroy(e);
    delete p;
}
void prof_enable(Prof *p, bool on) { p->on = on; }
bool prof_on(const Prof *p) { return p && p->on; }
// synchronise on the pending events, fold them into per-name totals
void prof_collect(Prof *p)
{
    for (auto &r : p->pending) {
        cudaEventSynchronize(r.b);
        float ms = 0;
        cudaEventElapsedTime(&ms, r.a, r.b);
        auto &x = p->acc[r.name];
        x.ms += ms;
        x.launches += 1;
        x.bfly += r.w.bfly;
        x.mac += r.w.mac;
        x.bytes += r.w.bytes;
        x.fbfly += r.w.fbfly;
        x.fmac += r.w.fmac;
        p->pool.push_back(r.a);
        p->pool.push_back(r.b);
    }
    p->pending.clear();
}
const std::map<std::string, ProfTotal> &prof_totals(Prof *p) { return p->acc; }
void prof_reset(Prof *p) { p->acc.clear(); }


namespace {

constexpr int COLS = 16;  // columns per column-phase CTA (16 x 8 B = one 128-B segment per row)

__host__ __device__ constexpr int b1_of(int log_n) { return log_n / 2; }

__device__ __forceinline__ const u64 *limb_ptr(const PolyMap &m, u32 p, u32 i, u32 log_n)
{
    return m.base + (((size_t)p * m.cap + i) << log_n);
}
__device__ __forceinline__ u64 *limb_ptr_w(const PolyMap &m, u32 p, u32 i, u32 log_n)
{
    return m.base + (((size_t)p * m.cap + i) << log_n);
}
__device__ __forceinline__ u32 prime_of(const LimbSet &ls, u32 i) { return i < ls.lq ? ls.qoff + i : ls.sp + (i - ls.lq); }

// ------------------------------------------------------------------------------------
// Column phase, forward (stages 0..B1-1).  One CTA = 16 adjacent columns of one limb.
// Task::get(r, src, dst, prime, src_prime) -> false means "skip this limb".
// ------------------------------------------------------------------------------------
struct TaskPlainCol {
    PolyMap src, dst;
    LimbSet ls;
    u32 log_n;
    FDiv fn{};  // division by ls.n (set by the launchers)
    int raw = 0;         // k_fwd_rows_store: FP64-mode limbs hold lazy doubles (k_fwd_cols_r16)
    __device__ bool get(u32 r, const u64 *&s, u64 *&d, u32 &prime, u32 &sprime) const
    {
        const u32 p = fn.m ? fn.div(r) : r / ls.n, i = r - p * ls.n;
        s = limb_ptr(src, p, i, log_n);
        d = limb_ptr_w(dst, p, i, log_n);
        prime = sprime = prime_of(ls, i);
        return true;
    }
};

struct TaskBcastCol {  // y[p][i] = NTT_{q_i}(X[p] mod q_i)
    const u64 *X;
    u64 *S;
    u32 nt, xprime, xstride, log_n, toff;
    FDiv fnt{};
    u32 lnt = 0, ltoff = 0;  // layout of S (a launch may cover a sub-range of its targets)
    // fused ModDown + rescale (reading A7): the source is the two-prime CRT value
    // X + q_last T (X < q_last, T < P; T dense [npolys][N]) reduced mod q_i as
    // [X]_{q_i} + [T]_{q_i} (q_last mod q_i), with qlc[i] = (q_last mod q_i, Shoup)
    const u64 *T = nullptr;
    const ulonglong2 *qlc = nullptr;
    // FP64-mode targets: [T]_{q_i} (q_{l-1} mod q_i) formed on the FP64 pipe from T's 31-bit halves,
    // qlcf[2i] = (c, c/q_i) with c = q_{l-1} mod q_i, qlcf[2i+1] = (2^31 c mod q_i, .../q_i)
    const double2 *qlcf = nullptr;
    __device__ const u64 *tsrc(u32 r) const { return T + (((size_t)(fnt.m ? fnt.div(r) : r / nt)) << log_n); }
    __device__ bool get(u32 r, const u64 *&s, u64 *&d, u32 &prime, u32 &sprime) const
    {
        const u32 p = fnt.m ? fnt.div(r) : r / nt, i = r - p * nt;
        s = X + (((size_t)p * xstride) << log_n);
        d = S + ((lnt ? (size_t)p * lnt + (toff + i - ltoff) : (size_t)r) << log_n);
        prime = toff + i;
        sprime = xprime;
        return true;
    }
};

// D layout: digit j of ciphertext c at ((j / dw) * dcnt + c0 + c) * dw + j % dw  (limbs) --
// [cnt][l] when dw = l (one rank), [R][count][w] after an all-gather of w-limb shards.
struct TaskModUpCol {  // I[c][tl][j] = cols(NTT_{q_t}(D[c][j] mod q_t)), j != t
    const u64 *D;
    u64 *I;
    u32 l, t0, T, sp, log_n, dw, dcnt, c0;
    FDiv fT{}, fl{};      // fl: division by the window's digit count nj
    u32 lt0 = 0, lT = 0;  // layout of I (a launch may cover a sub-range of its targets)
    u32 jw0 = 0, nj = 0;  // digit window [jw0, jw0 + nj) (pipelined limb sharding); nj = l: all
    __device__ bool get(u32 r, const u64 *&s, u64 *&d, u32 &prime, u32 &sprime) const
    {
        // target fastest in launch order: neighbouring CTAs use different primes, so integer-
        // and FP64-mode targets share the SMs (their pipes run concurrently)
        const u32 rest = fT.div(r), tl = r - rest * T, c = fl.div(rest), j = jw0 + (rest - c * nj);
        u32 t = t0 + tl;
        if (t == j) return false;
        s = D + ((((size_t)(j / dw) * dcnt + c0 + c) * dw + j % dw) << log_n);
        d = I + ((((size_t)c * (lT ? lT : T) + (lT ? t - lt0 : tl)) * l + j) << log_n);
        prime = (t < l) ? t : sp;
        sprime = j;
        return true;
    }
};

// PIPE: 0 = arithmetic mode chosen per prime at run time, 1 = FP64-mode primes only,
// 2 = integer-mode primes only (one code path -> fewer registers -> more resident CTAs)
template <int B1, int B2, class Task, int PIPE>
__device__ __forceinline__ void fwd_cols_body(const Task &task, const Tables &tb, u32 ngroups)
{
    __shared__ u64 sm[(1 << B1) * COLS];
    constexpr u32 log_n = B1 + B2, n2 = 1u << B2;  // compile-time strides: element offsets fold into the LD/ST
    const u32 lg = 31 - __clz(ngroups);  // ngroups is a power of two
    const u32 r = blockIdx.x >> lg, grp = blockIdx.x & (ngroups - 1);
    const int col = threadIdx.x % COLS, lt = threadIdx.x / COLS;
    const u64 *src;
    u64 *dst;
    u32 prime, sprime;
    if (!task.get(r, src, dst, prime, sprime)) return;
    const ModC m = load_mod(tb.mod, prime);
    const ulonglong2 *tw = tb.psi + ((size_t)prime << log_n);
    const bool f64 = PIPE == 1 ? true : PIPE == 2 ? false : use_f64(tb, m.q);
    // a residue mod a larger prime needs reducing mod q -- except in FP64 mode when the source
    // prime is below 2^42: the FP64 stages take any input < 2^50 and leave the result canonical
    const u64 qs = tb.mod[sprime].q;
    const bool red = f64 ? !use_f64(tb, qs) : qs > m.q;
    const u32 c = grp * COLS + col;
    const u64 *sp0 = src + (size_t)lt * n2 + c;  // element i at ((i << (B1-3)) | lt) * n2 + c
    u64 v[8];
    bool crt = false;
    if constexpr (std::is_same_v<Task, TaskBcastCol>) crt = task.T != nullptr;
    if constexpr (std::is_same_v<Task, TaskBcastCol> && PIPE == 1) {
        if (crt && task.qlcf) {  // FP64 pipe end to end: X + T_lo c + T_hi (2^31 c), |.| < 2^43
            const u64 *tp0 = task.tsrc(r) + (size_t)lt * n2 + c;
            const double2 *twf = tb.psif + ((size_t)prime << log_n);
            const double2 qq = __ldg(twf), c0 = __ldg(task.qlcf + 2 * prime), c1 = __ldg(task.qlcf + 2 * prime + 1);
            double d[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const size_t e = (size_t)i << (B1 - 3 + B2);
                const u64 tv = tp0[e];
                d[i] = u2d(sp0[e]) + f64_mulmod(u2d(tv & 0x7fffffffull), c0.x, c0.y, qq.x) +
                       f64_mulmod(u2d(tv >> 31), c1.x, c1.y, qq.x);
            }
            fwd_rounds_f64<B1, 0>(d, ColEx<COLS>{sm, col}, lt, 0, 0u, twf, qq.x);
            u64 *dp0 = dst + (size_t)(lt << 3) * n2 + c;
#pragma unroll
            for (int i = 0; i < 8; ++i) dp0[(size_t)i * n2] = f64_canon(d[i], qq.x, qq.y);
            return;
        }
    }
    if (crt) {  // (uniform per launch) two-prime CRT source of the fused ModDown + rescale
        if constexpr (std::is_same_v<Task, TaskBcastCol>) {
            const u64 *tp0 = task.tsrc(r) + (size_t)lt * n2 + c;
            const ulonglong2 qc = __ldg(task.qlc + prime);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const size_t e = (size_t)i << (B1 - 3 + B2);
                v[i] = addmod(reduce64(sp0[e], m.q, m.bar), shoup(reduce64(tp0[e], m.q, m.bar), qc.x, qc.y, m.q), m.q);
            }
        }
    } else if (red) {  // uniform per CTA: the reduction only runs where it is needed
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = reduce64(sp0[(size_t)i << (B1 - 3 + B2)], m.q, m.bar);
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = sp0[(size_t)i << (B1 - 3 + B2)];
    }
    if (std::is_same_v<Task, TaskModUpCol> && f64)  // ModUp slab: lazy doubles for the inner product
        fwd_tile_f64_raw<B1>(v, ColEx<COLS>{sm, col}, lt, 0, 0u, tb.psif + ((size_t)prime << log_n));
    else
        fwd_rounds<B1, 0>(v, ColEx<COLS>{sm, col}, lt, 0, 0u, tw, m.q, tb.psif + ((size_t)prime << log_n), f64);
    if (!f64 && lazy_wide<B1>(m.q)) {  // the row phase restarts from canonical values
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = reduce64(v[i], m.q, m.bar);
    }
    u64 *dp0 = dst + (size_t)(lt << 3) * n2 + c;  // element i at lidx(lt, i, 0) = 8 lt + i
#pragma unroll
    for (int i = 0; i < 8; ++i) dp0[(size_t)i * n2] = v[i];
}

template <int B1, int B2, class Task, int PIPE = 0>
__global__ void __launch_bounds__(COLS *(1 << B1) / 8) k_fwd_cols(Task task, Tables tb, u32 ngroups)
{
    fwd_cols_body<B1, B2, Task, PIPE>(task, tb, ngroups);
}
// FP64-only launches: the single code path fits 40 registers -> 1.5x the resident warps
template <int B1, int B2, class Task>
__global__ void __launch_bounds__(COLS *(1 << B1) / 8, 1536 / (COLS * (1 << B1) / 8))
    k_fwd_cols_f64(Task task, Tables tb, u32 ngroups)
{
    fwd_cols_body<B1, B2, Task, 1>(task, tb, ngroups);
}

// ------------------------------------------------------------------------------------
// Radix-16 FP64 ModUp column phase (FP64-mode targets; B1 >= 6).  16 adjacent columns per
// CTA, 2^(B1-4) threads per column (threadIdx = lt * 16 + col: every global access is a
// 128-byte segment), 16 values per thread: round 1 = global stages 0..3 on column-index bits
// B1-1..B1-4 (element li = (i << (B1-4)) | lt; their twiddles depend on i only), ONE shared-
// memory exchange, round 2 = stages 4..B1-1 (li = (lt << 4) | i).  Against the radix-8 tile of
// k_fwd_cols_f64: one exchange instead of two, 8 independent butterflies per stage per thread,
// and the slab left as lazy doubles (no canonicalisation: k_ks_mac CLS 5 continues from them).
// ------------------------------------------------------------------------------------
// One radix-16 CT stage on register bit P of 16 values: the pair (i, i | 2^P) (bit P clear) uses
// twiddle tw[i >> (P + 1)] (the caller offsets tw to the stage's run for this thread).
template <int P>
__device__ __forceinline__ void r16_stage(double d[16], const double2 *tw, double q)
{
    constexpr int bit = 1 << P;
#pragma unroll
    for (int e = 0; e < (16 >> (P + 1)); ++e) {
        const double2 w = __ldg(tw + e);
#pragma unroll
        for (int j = 0; j < bit; ++j) {
            const int i0 = (e << (P + 1)) | j, i1 = i0 | bit;
            const double t = f64_mulmod(d[i1], w.x, w.y, q);
            const double x = d[i0];
            d[i0] = x + t;
            d[i1] = x - t;
        }
    }
}

// Radix-16 FP64 forward column phase (every target / limb of the launch FP64-mode; B1 >= 6).
// 16 adjacent columns per CTA, 2^(B1-4) threads per column (threadIdx = lt * 16 + col: every
// global access is a 128-byte segment), 16 values per thread: round 1 = global stages 0..3 on
// column-index bits B1-1..B1-4 (element li = (i << (B1-4)) | lt; their twiddles depend on i
// only), ONE shared-memory exchange, round 2 = stages 4..B1-1 (li = (lt << 4) | i).  Against
// the radix-8 tile of k_fwd_cols_f64: one exchange instead of two and 8 independent butterflies
// per stage per thread; the output is left as lazy doubles (|v| < 2^46, no canonicalisation)
// for the row-phase kernel that continues from it (k_ks_mac CLS 5 for the ModUp slabs,
// k_fwd_rows_submul with s_raw for the broadcast, k_fwd_rows_store with raw).
//   TaskModUpCol: digit D_j mod q_t (diagonal tiles skipped);  TaskBcastCol: the rescale /
//   ModDown source (or the fused two-prime CRT value) reduced into q_t;  TaskPlainCol /
//   TaskHybSlot: a canonical limb in place.
template <class Task>
__device__ __forceinline__ void r16_load(const Task &task, const Tables &tb, u32 r, const u64 *src, u32 prime,
                                         u32 sprime, size_t off, size_t rs, double q, double d[16])
{
    const u64 *sp0 = src + off;
    if constexpr (std::is_same_v<Task, TaskBcastCol>) {
        if (task.T) {  // X + T_lo c + T_hi (2^31 c) on the FP64 pipe, |.| < 2^44
            const u64 *tp0 = task.tsrc(r) + off;
            const double2 c0 = __ldg(task.qlcf + 2 * prime), c1 = __ldg(task.qlcf + 2 * prime + 1);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const u64 tv = tp0[(size_t)i * rs];
                d[i] = u2d(sp0[(size_t)i * rs]) + f64_mulmod(u2d(tv & 0x7fffffffull), c0.x, c0.y, q) +
                       f64_mulmod(u2d(tv >> 31), c1.x, c1.y, q);
            }
            return;
        }
    }
    if (!use_f64(tb, __ldg(&tb.mod[sprime].q))) {  // source prime >= 2^42: reduce mod q_t first
        const ModC m = load_mod(tb.mod, prime);
#pragma unroll
        for (int i = 0; i < 16; ++i) d[i] = u2d(reduce64(sp0[(size_t)i * rs], m.q, m.bar));
    } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) d[i] = u2d(sp0[(size_t)i * rs]);
    }
}

template <int B1, int B2, class Task>
__global__ void __launch_bounds__(1 << B1) k_fwd_cols_r16(Task task, Tables tb, u32 ngroups)
{
    static_assert(B1 >= 6 && B1 <= 8, "radix-16 column tile");
    __shared__ double sm[(1 << B1) * 16];
    constexpr u32 log_n = B1 + B2, n2 = 1u << B2;
    const u32 r = blockIdx.x >> (31 - __clz(ngroups)), grp = blockIdx.x & (ngroups - 1);
    const int col = threadIdx.x & 15, lt = threadIdx.x >> 4;
    const u64 *src;
    u64 *dst;
    u32 prime, sprime;
    if (!task.get(r, src, dst, prime, sprime)) return;
    if (!use_f64(tb, __ldg(&tb.mod[prime].q))) return;  // (uniform per CTA; launches are class-filtered)
    const double2 *twf = tb.psif + ((size_t)prime << log_n);
    const double2 qq = __ldg(twf);
    const double q = qq.x;
    const u32 c = grp * 16 + col;
    double d[16];
    r16_load(task, tb, r, src, prime, sprime, (size_t)lt * n2 + c, (size_t)1 << (B1 - 4 + B2), q, d);
    r16_stage<3>(d, twf + 1, q);
    r16_stage<2>(d, twf + 2, q);
    r16_stage<1>(d, twf + 4, q);
    r16_stage<0>(d, twf + 8, q);
    // (in-place tasks: every global load of the CTA precedes the exchange barrier, hence any store)
#pragma unroll
    for (int i = 0; i < 16; ++i) sm[((i << (B1 - 4)) | lt) * 16 + col] = d[i];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 16; ++i) d[i] = sm[((lt << 4) | i) * 16 + col];
    if constexpr (B1 >= 5) r16_stage<B1 - 5>(d, twf + (1u << 4) + ((u32)lt << (3 - (B1 - 5))), q);
    if constexpr (B1 >= 6) r16_stage<B1 - 6>(d, twf + (1u << 5) + ((u32)lt << (3 - (B1 - 6))), q);
    if constexpr (B1 >= 7) r16_stage<B1 - 7>(d, twf + (1u << 6) + ((u32)lt << (3 - (B1 - 7))), q);
    if constexpr (B1 >= 8) r16_stage<B1 - 8>(d, twf + (1u << 7) + ((u32)lt << (3 - (B1 - 8))), q);
    u64 *dp0 = dst + (size_t)(lt << 4) * n2 + c;  // element li = (lt << 4) | i
#pragma unroll
    for (int i = 0; i < 16; ++i) dp0[(size_t)i * n2] = (u64)__double_as_longlong(d[i]);
}

// One radix-16 Gentleman-Sande stage on register bit P: (x, y) = (d[i], d[i | 2^P]) ->
// (x + y, (x - y) w) with w = tw[i >> (P + 1)].
template <int P>
__device__ __forceinline__ void r16_gs_stage(double d[16], const double2 *tw, double q)
{
    constexpr int bit = 1 << P;
#pragma unroll
    for (int e = 0; e < (16 >> (P + 1)); ++e) {
        const double2 w = __ldg(tw + e);
#pragma unroll
        for (int j = 0; j < bit; ++j) {
            const int i0 = (e << (P + 1)) | j, i1 = i0 | bit;
            const double x = d[i0], y = d[i1];
            d[i0] = x + y;
            d[i1] = f64_mulmod(x - y, w.x, w.y, q);
        }
    }
}

// Radix-16 FP64 inverse column phase (plain INTT, FP64-mode limbs), in place on the row-phase
// output: round 1 = GS stages on column-index bits 0..3 (li = (lt << 4) | i; twiddle runs per
// thread), one exchange, round 2 = bits 4..B1-1 (li = (i << (B1-4)) | lt; runs uniform), then
// N^{-1} and the canonical residue.  (Sums grow 16x per round: reduced once between rounds.)
// CC columns per CTA (16: every global access a 128-byte segment; 8: twice the CTAs for launches
// of a few dozen limbs, which would otherwise fill less than one wave)
template <int B1, int B2, int CC = 16>
__global__ void __launch_bounds__(CC << (B1 - 4), 1024 / (CC << (B1 - 4))) k_inv_cols_r16(TaskPlainCol task, Tables tb, u32 ngroups)
{
    __shared__ double sm[(1 << B1) * CC];
    constexpr u32 log_n = B1 + B2, n2 = 1u << B2;
    const u32 r = blockIdx.x >> (31 - __clz(ngroups)), grp = blockIdx.x & (ngroups - 1);
    const int col = threadIdx.x % CC, lt = threadIdx.x / CC;
    const u64 *src;
    u64 *dst;
    u32 prime, sprime;
    task.get(r, src, dst, prime, sprime);
    const double2 *itw = tb.ipsif + ((size_t)prime << log_n);
    const double2 qq = __ldg(itw);
    const double q = qq.x;
    const u32 c = grp * CC + col;
    double d[16];
    const u64 *lp0 = dst + (size_t)(lt << 4) * n2 + c;  // element li = (lt << 4) | i (in place)
#pragma unroll
    for (int i = 0; i < 16; ++i) d[i] = u2d(lp0[(size_t)i * n2]);
    // GS stage on bit qq of li uses twiddle 2^(B1-1-qq) + (li >> (qq + 1))
    r16_gs_stage<0>(d, itw + (1u << (B1 - 1)) + ((u32)lt << 3), q);
    r16_gs_stage<1>(d, itw + (1u << (B1 - 2)) + ((u32)lt << 2), q);
    r16_gs_stage<2>(d, itw + (1u << (B1 - 3)) + ((u32)lt << 1), q);
    r16_gs_stage<3>(d, itw + (1u << (B1 - 4)) + (u32)lt, q);
#pragma unroll
    for (int i = 0; i < 16; ++i) sm[((lt << 4) | i) * CC + col] = f64_red(d[i], q, qq.y);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 16; ++i) d[i] = sm[((i << (B1 - 4)) | lt) * CC + col];
    // bit qq = 4..B1-1 is register bit P = qq - (B1 - 4); run 2^(B1-1-qq)
    if constexpr (B1 >= 5) r16_gs_stage<8 - B1>(d, itw + (1u << (B1 - 5)), q);
    if constexpr (B1 >= 6) r16_gs_stage<9 - B1>(d, itw + (1u << (B1 - 6)), q);
    if constexpr (B1 >= 7) r16_gs_stage<10 - B1>(d, itw + (1u << (B1 - 7)), q);
    if constexpr (B1 >= 8) r16_gs_stage<11 - B1>(d, itw + (1u << (B1 - 8)), q);
    const ulonglong2 ni = __ldg(tb.ninv + prime);
    const double nf = u2d(ni.x), nfq = nf * qq.y;
    u64 *sp0 = dst + (size_t)lt * n2 + c;  // element li = (i << (B1-4)) | lt
#pragma unroll
    for (int i = 0; i < 16; ++i) sp0[(size_t)i << (B1 - 4 + B2)] = f64_canon(f64_mulmod(d[i], nf, nfq, q), q, qq.y);
}

template <int B1, int B2>
void inv_cols_r16_launch(const Launch &L, const TaskPlainCol &t, u32 nlimbs, const Work &w)
{
    constexpr int B1e = B1 >= 6 ? B1 : 6;
    const u32 g16 = (1u << B2) / 16;
    if ((size_t)nlimbs * g16 < (size_t)L.n_sm * 8) {  // under two waves of 16-column CTAs: 8 columns
        const u32 g8 = (1u << B2) / 8;
        KLAUNCH(L, "ntt_inv_cols", w, (k_inv_cols_r16<B1e, B2, 8><<<nlimbs * g8, 8 << (B1e - 4), 0, L.st>>>(t, *L.tb, g8)));
    } else {
        KLAUNCH(L, "ntt_inv_cols", w, (k_inv_cols_r16<B1e, B2, 16><<<nlimbs * g16, 16 << (B1e - 4), 0, L.st>>>(t, *L.tb, g16)));
    }
}

// ------------------------------------------------------------------------------------
// Row phase, forward (stages B1..logN-1).  A row (2^B2 contiguous words) per
// THR = 2^B2/8 threads, R rows per CTA; warp-synchronous.
// ------------------------------------------------------------------------------------
template <int B2>
struct RowGeom {
    static constexpr int THR = (1 << B2) / 8;
    static constexpr int R = 128 / THR;                  // rows per CTA (128 threads)
    static constexpr int SROW = (1 << B2) + (1 << B2) / 16;  // padded row in smem
};

// load the row in forward-first layout: li = (i << (B2-3)) | lt
template <int B2>
__device__ __forceinline__ void load_row_fwd(u64 v[8], const u64 *row, int lt)
{
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = row[(i << (B2 - 3)) | lt];
}

// thread-contiguous 8 words (li = 8 lt + i), 16-byte vector accesses
__device__ __forceinline__ void load8(u64 v[8], const u64 *p)
{
    const ulonglong2 *q = reinterpret_cast<const ulonglong2 *>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        ulonglong2 x = q[i];
        v[2 * i] = x.x;
        v[2 * i + 1] = x.y;
    }
}
__device__ __forceinline__ void load8_stream(u64 v[8], const u64 *p)
{
    const ulonglong2 *q = reinterpret_cast<const ulonglong2 *>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        ulonglong2 x = __ldcs(q + i);
        v[2 * i] = x.x;
        v[2 * i + 1] = x.y;
    }
}
__device__ __forceinline__ void store8(u64 *p, const u64 v[8])
{
    ulonglong2 *q = reinterpret_cast<ulonglong2 *>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) q[i] = make_ulonglong2(v[2 * i], v[2 * i + 1]);
}

template <int B2, class Task>
__global__ void __launch_bounds__(128) k_fwd_rows_store(Task task, Tables tb, u32 ngroups)
{
    using G = RowGeom<B2>;
    __shared__ u64 sm[G::R * G::SROW];
    const u32 log_n = tb.log_n;
    const u32 B1 = log_n - B2;
    const u32 r = blockIdx.x >> (31 - __clz(ngroups)), grp = blockIdx.x & (ngroups - 1);
    const int rin = threadIdx.x / G::THR, lt = threadIdx.x % G::THR;
    const u32 row = grp * G::R + rin;
    const u64 *src;
    u64 *dst;
    u32 prime, sprime;
    if (!task.get(r, src, dst, prime, sprime)) return;
    const ModC m = load_mod(tb.mod, prime);
    const ulonglong2 *tw = tb.psi + ((size_t)prime << log_n);
    const bool f64 = use_f64(tb, m.q);
    u64 v[8];
    load_row_fwd<B2>(v, src + ((size_t)row << B2), lt);
    const RowEx ex{sm + rin * G::SROW};
    if (f64 && task.raw) {  // lazy doubles from k_fwd_cols_r16
        const double2 *twf = tb.psif + ((size_t)prime << log_n);
        const double2 qq = __ldg(twf);
        double d[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) d[i] = __longlong_as_double((long long)v[i]);
        fwd_rounds_f64<B2, 0>(d, ex, lt, B1, row, twf, qq.x);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = f64_canon(d[i], qq.x, qq.y);
    } else {
        fwd_rounds<B2, 0>(v, ex, lt, B1, row, tw, m.q, tb.psif + ((size_t)prime << log_n), f64);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = fwd_canon<B2>(v[i], m, f64);
    }
    ex(v, lt, 0, B2 - 3);  // to the coalesced layout li = (i << (B2-3)) | lt
    u64 *drow = dst + ((size_t)row << B2);
#pragma unroll
    for (int i = 0; i < 8; ++i) drow[(i << (B2 - 3)) | lt] = v[i];
}

// rescale / ModDown epilogue: out = [base] + (x - y) * C_i
struct SubMulArgs {
    const u64 *S;  // [npolys][nt][N] phase-1 outputs
    u32 nt, toff;  // targets toff .. toff + nt - 1 (global limb indices)
    PolyMap x, out, base;
    PolyMap acc;   // optional second addend read at the output index (TotalSum: ct += rot(ct))
    const u32 *base_perm;
    int base_c0_only;
    const ulonglong2 *consts;
    const ulonglong2 *bconsts = nullptr;  // base scaled by bconsts[i] (fused ModDown + rescale)
    int s_raw = 0;  // FP64-mode targets' S rows hold lazy doubles (k_fwd_cols_r16)
};

template <int B2>
__global__ void __launch_bounds__(128) k_fwd_rows_submul(SubMulArgs a, Tables tb, u32 ngroups)
{
    using G = RowGeom<B2>;
    __shared__ u64 sm[G::R * G::SROW];
    const u32 log_n = tb.log_n;
    const u32 B1 = log_n - B2;
    const u32 r = blockIdx.x >> (31 - __clz(ngroups)), grp = blockIdx.x & (ngroups - 1);
    const int rin = threadIdx.x / G::THR, lt = threadIdx.x % G::THR;
    const u32 row = grp * G::R + rin;
    const u32 p = r / a.nt, i = a.toff + r % a.nt;  // global limb / prime index
    const ModC m = load_mod(tb.mod, i);
    const ulonglong2 *tw = tb.psi + ((size_t)i << log_n);
    const bool f64 = use_f64(tb, m.q);
    u64 v[8];
    load_row_fwd<B2>(v, a.S + ((size_t)r << log_n) + ((size_t)row << B2), lt);
    const RowEx ex{sm + rin * G::SROW};
    if (f64 && a.s_raw) {  // lazy doubles from the radix-16 broadcast columns
        const double2 *twf = tb.psif + ((size_t)i << log_n);
        const double2 qq = __ldg(twf);
        double d[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) d[k] = __longlong_as_double((long long)v[k]);
        fwd_rounds_f64<B2, 0>(d, ex, lt, B1, row, twf, qq.x);
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = f64_canon(d[k], qq.x, qq.y);
    } else {
        fwd_rounds<B2, 0>(v, ex, lt, B1, row, tw, m.q, tb.psif + ((size_t)i << log_n), f64);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = fwd_canon<B2>(v[k], m, f64);
    ex(v, lt, 0, B2 - 3);  // epilogue in the coalesced layout: element k at (k << (B2-3)) | lt
    const u32 roff = row << B2;
    const u64 *xp = limb_ptr(a.x, p, i, log_n) + roff;
    const ulonglong2 c = __ldg(a.consts + i);
    u64 o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = shoup(xp[(k << (B2 - 3)) | lt] + m.q - v[k], c.x, c.y, m.q);
    if (a.base.base != nullptr && (!a.base_c0_only || (p & 1) == 0)) {
        const u64 *bp = limb_ptr(a.base, p, i, log_n);
        if (a.base_perm) {
#pragma unroll
            for (int k = 0; k < 8; ++k) o[k] = addmod(o[k], bp[__ldg(a.base_perm + roff + ((k << (B2 - 3)) | lt))], m.q);
        } else if (a.bconsts) {
            const ulonglong2 bc = __ldg(a.bconsts + i);
#pragma unroll
            for (int k = 0; k < 8; ++k) o[k] = addmod(o[k], shoup(bp[roff + ((k << (B2 - 3)) | lt)], bc.x, bc.y, m.q), m.q);
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) o[k] = addmod(o[k], bp[roff + ((k << (B2 - 3)) | lt)], m.q);
        }
    }
    if (a.acc.base != nullptr) {
        const u64 *ap = limb_ptr(a.acc, p, i, log_n) + roff;
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = addmod(o[k], ap[(k << (B2 - 3)) | lt], m.q);
    }
    u64 *op = limb_ptr_w(a.out, p, i, log_n) + roff;
#pragma unroll
    for (int k = 0; k < 8; ++k) op[(k << (B2 - 3)) | lt] = o[k];
}

// ------------------------------------------------------------------------------------
// Key switch inner product: for target t and each digit j, finish the forward NTT of
// (D_j mod q_t) (row phase) and multiply-accumulate with the key in 128 bits; the
// key streams from HBM exactly once, the accumulators never leave registers.
// ------------------------------------------------------------------------------------
struct MacArgs {
    const u64 *I;
    PolyMap din;
    const u32 *perm;
    const u64 *key;
    u64 *ext;
    u32 Lk, l, t0, T, sp;
    u32 t0i, Ti;  // target range of the I layout (I[c][t - t0i][j], Ti targets per ciphertext)
    FDiv fT{};    // division by T (set in mac_launch)
    // digit-split mode (part != nullptr): CTA row blockIdx.y sums digits [y*jper, (y+1)*jper)
    // into part[y][c][0|1][t - t0] (canonical); k_ks_split_sum adds the partial sums into ext
    u64 *part = nullptr;
    u32 jper = 0, cnt_run = 0;
    // ModDown fusion: the special-prime target's rows leave with the INTT row phase already
    // applied (the accumulator's first inverse stages; the ModDown continues with the columns)
    int pinv_rows = 0;
    // digit window [jw0, jw1) (pipelined limb sharding; jw1 = 0: all l digits) and accumulate
    // mode: the window's sum is added mod q_t to the ext value already there
    u32 jw0 = 0, jw1 = 0;
    int accum = 0;
    int kcomp = 0;  // FP64 class: key rows compact (launch_key_compact)
    // hybrid mode (halpha > 0, CLS 5 only): digits of halpha limbs, nd = beta of them; target t is
    // an extended slot (t < l: q_t, t = l + k: special p_k = prime sp + k, key limb Lk + k); the
    // row-phase input is X[c][d][t] (layout [cnt][nd][next][N], hyb_ntt_impl's column output),
    // the diagonal digit of a slot t < l is t / halpha; key [nd][2][kst][N]; ext [cnt][2][next][N]
    u32 halpha = 0, nd = 0, next = 0, kst = 0;
    // fused hybrid ModDown + rescale (launch_hyb_moddown_rs, rows done here): targets t >= l-1 leave
    // with the INTT row phase applied, t = l-1 after z = P base_{l-1} + acc_{l-1} (zrs[l-1] = P mod q)
    int rs_rows = 0;
    PolyMap zbase{};
    const ulonglong2 *zrs = nullptr;
};

template <int B2>
struct MacGeom {
    static constexpr int THR = (1 << B2) / 8;   // threads per row
    static constexpr int R = 64 / THR;          // rows per CTA (64 threads)
    static constexpr int ROW = 1 << B2;         // words per row
    static constexpr int SROW = ROW + ROW / 16; // padded exchange row
    static constexpr int STAGE = 3 * ROW;       // per row per pipeline stage: I (or d), key b, key a
    static constexpr int CH = ROW / 2 / THR;    // 16-byte chunks per thread per array
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

// key chunk c (16 B) of row rin lives at chunk slot kswz(c, rin): threads read chunks
// 4lt..4lt+3 (their 8 contiguous words) -- conflict-free for every B2
// compact key low plane: 16-byte chunk c (4 residues) at slot c ^ ((c >> 3) & 1): a quarter-warp's
// 8 lanes read chunks 2 lt (+1), i.e. 8 distinct bank groups
__device__ __forceinline__ int kc_lo_swz(int c) { return c ^ ((c >> 3) & 1); }
// diagonal digit row in the inner-product pipeline: 16-byte chunk c at slot c ^ ((c >> 3) & 7), so
// the 8 lanes of a quarter-warp reading elements 8 lt .. 8 lt + 7 (chunks 4 lt .. 4 lt + 3) hit 8
// distinct bank groups (natural layout: 4-way conflicts, ncu profiles/ncu_r2_c4_k_ks_mac.txt)
__device__ __forceinline__ int dg_cswz(int c) { return c ^ ((c >> 3) & 7); }
__device__ __forceinline__ int dg_swz(int e) { return 2 * dg_cswz(e >> 1) + (e & 1); }
__device__ __forceinline__ int kswz(int c, int rin) { return (c & ~7) | ((c ^ ((c >> 3) + 2 * rin)) & 7); }

// One CTA = R rows of one (ciphertext, target).  Digit loop software-pipelined: the next
// digit's phase-1 row and both key rows stream into shared memory with cp.async while
// the current digit's row-phase NTT and 128-bit multiply-accumulate run.
template <int B2, class Acc, bool LAZY>
__device__ __forceinline__ void ks_mac_body(const MacArgs &a, const Tables &tb, u32 ngroups,
                                            u64 (*buf)[MacGeom<B2>::R][MacGeom<B2>::STAGE], u64 *sx)
{
    using G = MacGeom<B2>;
    const u32 log_n = tb.log_n;
    const u32 B1 = log_n - B2;
    const u32 cr = blockIdx.x >> (31 - __clz(ngroups)), grp = blockIdx.x & (ngroups - 1);  // cr = c * T + tl
    const u32 c = a.fT.div(cr), tl = cr - c * a.T;
    const u32 t = a.t0 + tl;
    const u32 ct = c * a.Ti + (t - a.t0i);  // slab index in the I layout
    const int rin = threadIdx.x / G::THR, lt = threadIdx.x % G::THR;
    const u32 row = grp * G::R + rin;
    const u32 prime = (t < a.l) ? t : a.sp;
    const u32 klimb = (t < a.l) ? t : a.Lk;
    const ModC m = load_mod(tb.mod, prime);
    const ulonglong2 *tw = tb.psi + ((size_t)prime << log_n);
    const size_t nn = (size_t)1 << log_n;
    const u32 roff = row << B2;
    const u64 *dp = limb_ptr(a.din, c, t < a.l ? t : 0, log_n);

    auto issue = [&](u32 j, int s) {
        u64 *sI = buf[s][rin], *sb = sI + G::ROW, *sa = sb + G::ROW;
        const u64 *kb = a.key + ((size_t)(2 * j) * (a.Lk + 1) + klimb) * nn + roff;
        const u64 *ka = kb + (size_t)(a.Lk + 1) * nn;
        if (j == t) {
            if (a.perm) {
#pragma unroll
                for (int i = 0; i < 8; ++i) cp_async8(sI + 8 * lt + i, dp + __ldg(a.perm + roff + 8 * lt + i));
            } else {
#pragma unroll
                for (int k = 0; k < G::CH; ++k) {
                    const int ch = lt + G::THR * k;
                    cp_async16(sI + 2 * ch, dp + roff + 2 * ch);
                }
            }
        } else {
            const u64 *ip = a.I + ((((size_t)ct * a.l) + j) << log_n) + roff;
#pragma unroll
            for (int k = 0; k < G::CH; ++k) {
                const int ch = lt + G::THR * k;
                cp_async16(sI + 2 * ch, ip + 2 * ch);
            }
        }
#pragma unroll
        for (int k = 0; k < G::CH; ++k) {
            const int ch = lt + G::THR * k;
            cp_async16(sb + 2 * kswz(ch, rin), kb + 2 * ch);
            cp_async16(sa + 2 * kswz(ch, rin), ka + 2 * ch);
        }
    };

    const u32 jwe = a.jw1 ? a.jw1 : a.l;
    const u32 j0 = a.jw0 + (a.part ? blockIdx.y * a.jper : 0), j1 = a.part ? min(jwe, j0 + a.jper) : jwe;
    Acc acc0[8], acc1[8];
    issue(j0, 0);
    cp_async_commit();
    for (u32 j = j0; j < j1; ++j) {
        const int s = (j - j0) & 1;
        if (j + 1 < j1) issue(j + 1, s ^ 1);
        cp_async_commit();
        cp_async_wait1();
        __syncwarp();
        const u64 *sI = buf[s][rin], *sb = sI + G::ROW, *sa = sb + G::ROW;
        u64 v[8];
        if (j == t) {
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = sI[8 * lt + k];
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = sI[(k << (B2 - 3)) | lt];
            fwd_rounds_t<B2, 0, LAZY>(v, RowEx{sx + rin * G::SROW}, lt, B1, row, tw, m.q);
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = LAZY ? reduce64(v[k], m.q, m.bar) : csub(csub(v[k], 2 * m.q), m.q);
        }
        u64 wb[8], wa[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(sb + 2 * kswz(4 * lt + k, rin));
            const ulonglong2 y = *reinterpret_cast<const ulonglong2 *>(sa + 2 * kswz(4 * lt + k, rin));
            wb[2 * k] = x.x;
            wb[2 * k + 1] = x.y;
            wa[2 * k] = y.x;
            wa[2 * k + 1] = y.y;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            acc0[k].mac(v[k], wb[k]);
            acc1[k].mac(v[k], wa[k]);
        }
        __syncwarp();  // everyone done reading stage s before it is refilled
    }
    u64 o0[8], o1[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        o0[k] = acc0[k].reduce(m);
        o1[k] = acc1[k].reduce(m);
    }
    const RowEx ex{sx + rin * G::SROW};  // coalesced stores: element k at (k << (B2-3)) | lt
    ex(o0, lt, 0, B2 - 3);
    ex(o1, lt, 0, B2 - 3);
    u64 *e0 = a.part ? a.part + ((((size_t)blockIdx.y * a.cnt_run + c) * 2 * a.T + tl) << log_n) + roff
                     : a.ext + (((size_t)c * 2 * (a.l + 1) + t) << log_n) + roff;
    u64 *e1 = e0 + ((size_t)(a.part ? a.T : a.l + 1) << log_n);
    if (a.accum) {  // digit window after the first: add to the windows summed so far
        const u64 qa = __ldg(&tb.mod[(t < a.l) ? t : a.sp].q);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            e0[(k << (B2 - 3)) | lt] = addmod(o0[k], e0[(k << (B2 - 3)) | lt], qa);
            e1[(k << (B2 - 3)) | lt] = addmod(o1[k], e1[(k << (B2 - 3)) | lt], qa);
        }
        return;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        e0[(k << (B2 - 3)) | lt] = o0[k];
        e1[(k << (B2 - 3)) | lt] = o1[k];
    }
}

// FP64-pipe key switch (CLS 5, q_t < tb.f64_qmax): the row-phase NTT leaves each value a
// lazy signed double (|v| < 11.5q), and the inner product runs on the FP64 pipe too:
// r = v k - round(v k / q) q is formed exactly (FMA two-product, ntt.cuh f64_mulmod with the
// quotient taken from the rounded product), |r| < 2.5q, and summed in a double accumulator
// (|acc| < 2.5 l q < 2^50 for l <= 64, exact); one f64_canon per output.  Replaces the
// 128-bit integer accumulators (~18 integer instructions per MAC plus a ~30-instruction
// reduce128 per output) with 7 FP64 operations per MAC -- the integer issue slots were this
// kernel's bound (profiles/ncu_r1_v6_k_ks_mac.txt).
__device__ __forceinline__ double f64_mac_term(double v, double k, double q, double qinv)
{
    const double h = v * k;
    const double l = fma(v, k, -h);
    const double c = fma(h, qinv, F64_C) - F64_C;
    return fma(-c, q, h) + l;
}

__host__ __device__ constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c(x / 2); }

// Shared memory: a double-buffered phase-1 row (the next digit's row streams in while the
// current one is transformed) and ONE key stage: the next digit's key rows are issued right
// after this digit's multiply-accumulate and waited for only after the next transform, so the
// transform hides their latency.  20 KB per CTA instead of 29 KB -> 10 CTAs (20 warps) per SM.
template <int B2>
__device__ __forceinline__ void ks_mac_body_f64(const MacArgs &a, const Tables &tb, u32 ngroups,
                                                u64 (*sI)[MacGeom<B2>::R][MacGeom<B2>::SROW],
                                                u64 (*sk)[2 * MacGeom<B2>::ROW], double2 *tws, u32 tile)
{
    using G = MacGeom<B2>;
    const u32 log_n = tb.log_n;
    const u32 B1 = log_n - B2;
    const u32 cr = tile >> (31 - __clz(ngroups)), grp = tile & (ngroups - 1);
    const u32 c = a.fT.div(cr), tl = cr - c * a.T;
    const u32 t = a.t0 + tl;
    const u32 ct = c * a.Ti + (t - a.t0i);
    const int rin = threadIdx.x / G::THR, lt = threadIdx.x % G::THR;
    const u32 row = grp * G::R + rin;
    const u32 prime = (t < a.l) ? t : a.sp + (t - a.l);
    const u32 klimb = (t < a.l) ? t : a.Lk + (t - a.l);
    const u32 nd = a.halpha ? a.nd : a.l, next = a.halpha ? a.next : a.l + 1, kst = a.halpha ? a.kst : a.Lk + 1;
    const u32 tdiag = a.halpha ? (t < a.l ? t / a.halpha : 0xffffffffu) : t;  // the digit that holds t itself
    const double2 *twf = tb.psif + ((size_t)prime << log_n);
    const double2 qq = __ldg(twf);  // entry 0: (q, 1/q)
    const size_t nn = (size_t)1 << log_n;
    const u32 roff = row << B2;
    const u64 *dp = limb_ptr(a.din, c, t < a.l ? t : 0, log_n);
    u64 *skb = sk[rin], *ska = skb + G::ROW;
    // Row-phase twiddles of this CTA's R rows, cached in shared memory once and reused by every
    // digit (they depend on the target and the rows only): stage s of row rin needs the 2^s
    // entries at 2^(B1+s) + row 2^s ...; the cache keeps them at R 2^s + rin 2^s ..., i.e. the
    // ntt.cuh index formula with k = log2 R and hi = rin.  (From L2 they were the kernel's top
    // long-scoreboard stall: ncu profiles/ncu_r1_v7_k_ks_mac.txt.)
    constexpr int LOGR = ilog2c(G::R);
    static_assert((1 << LOGR) == G::R, "rows per CTA is a power of two");
    {  // each warp fills its own rows' entries (so a __syncwarp publishes them)
        constexpr int RPW = 32 / G::THR;  // rows per warp
        const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
        for (int st = 0; st < B2; ++st) {
            const int cnt = RPW << st;
            const double2 *src = twf + (1u << (B1 + st)) + ((size_t)(grp * G::R + w * RPW) << st);
            double2 *dst = tws + (G::R << st) + ((w * RPW) << st);
            for (int e = lane; e < cnt; e += 32) cp_async16(dst + tw_cache_swz((u32)(((w * RPW) << st) + e), st) - ((w * RPW) << st), src + e);
        }
    }

    auto issue_row = [&](u32 j, int s) {
        u64 *d = sI[s][rin];
        if (j == tdiag) {
            if (a.perm) {
#pragma unroll
                for (int i = 0; i < 8; ++i) cp_async8(d + dg_swz(8 * lt + i), dp + __ldg(a.perm + roff + 8 * lt + i));
            } else {
#pragma unroll
                for (int k = 0; k < G::CH; ++k) {
                    const int ch = lt + G::THR * k;
                    cp_async16(d + 2 * dg_cswz(ch), dp + roff + 2 * ch);
                }
            }
        } else {
            const u64 *ip = a.I + (a.halpha ? ((((size_t)c * nd + j) * next + t) << log_n)
                                            : ((((size_t)ct * a.l) + j) << log_n)) + roff;
#pragma unroll
            for (int k = 0; k < G::CH; ++k) {
                const int ch = lt + G::THR * k;
                cp_async16(d + 2 * ch, ip + 2 * ch);
            }
        }
    };
    auto issue_key = [&](u32 j) {
        const u64 *kb = a.key + ((size_t)(2 * j) * kst + klimb) * nn + roff;
        const u64 *ka = kb + (size_t)kst * nn;
        if (a.kcomp) {  // u32 low plane at the row slot, u8 high plane after N u32 (kc_* below)
            const unsigned char *rb = reinterpret_cast<const unsigned char *>(kb - roff);
            const unsigned char *ra = reinterpret_cast<const unsigned char *>(ka - roff);
            unsigned char *sb = reinterpret_cast<unsigned char *>(skb);
#pragma unroll
            for (int k = 0; k < G::ROW / 4 / G::THR; ++k) {  // low planes: ROW/4 chunks each
                const int ch = lt + G::THR * k;
                cp_async16(sb + 16 * kc_lo_swz(ch), rb + 4 * roff + 16 * ch);
                cp_async16(sb + 4 * G::ROW + 16 * kc_lo_swz(ch), ra + 4 * roff + 16 * ch);
            }
            if (lt < G::ROW / 16) {  // high planes: ROW/16 chunks each
                cp_async16(sb + 8 * G::ROW + 16 * lt, rb + 4 * nn + roff + 16 * lt);
                cp_async16(sb + 9 * G::ROW + 16 * lt, ra + 4 * nn + roff + 16 * lt);
            }
            return;
        }
#pragma unroll
        for (int k = 0; k < G::CH; ++k) {
            const int ch = lt + G::THR * k;
            cp_async16(skb + 2 * kswz(ch, rin), kb + 2 * ch);
            cp_async16(ska + 2 * kswz(ch, rin), ka + 2 * ch);
        }
    };

    double acc0[8], acc1[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc0[k] = acc1[k] = 0.0;
    // commit groups, in order: row_0, key_0, then per digit j: row_{j+1}, key_{j+1}
    const u32 jwe = a.jw1 ? a.jw1 : nd;
    const u32 j0 = a.jw0 + (a.part ? blockIdx.y * a.jper : 0), j1 = a.part ? min(jwe, j0 + a.jper) : jwe;
    issue_row(j0, 0);
    cp_async_commit();
    issue_key(j0);
    cp_async_commit();
    for (u32 j = j0; j < j1; ++j) {
        const int s = (j - j0) & 1;
        if (j + 1 < j1) issue_row(j + 1, s ^ 1);
        cp_async_commit();
        asm volatile("cp.async.wait_group 2;\n" ::);  // row_j landed (key_j, row_{j+1} may pend)
        __syncwarp();
        double v[8];
        if (j == tdiag) {
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = u2d(sI[s][rin][dg_swz(8 * lt + k)]);
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = __longlong_as_double((long long)sI[s][rin][(k << (B2 - 3)) | lt]);
            // (the ModUp slab holds lazy doubles |v| < 2^44: the row phase continues from them)
            // the row stage is free once loaded (refilled only next iteration): exchange buffer
            fwd_rounds_f64<B2, 0, RowEx, true>(v, RowEx{sI[s][rin]}, lt, LOGR, (u32)rin, tws, qq.x);
        }
        cp_async_wait1();  // key_j landed (row_{j+1} may pend)
        __syncwarp();
        if (a.kcomp) {  // elements 8 lt .. 8 lt + 7: two low-plane chunks + 8 high bytes per polynomial
            const unsigned char *sb = reinterpret_cast<const unsigned char *>(skb);
#pragma unroll
            for (int p2 = 0; p2 < 2; ++p2) {
                const uint4 l0 = *reinterpret_cast<const uint4 *>(sb + p2 * 4 * G::ROW + 16 * kc_lo_swz(2 * lt));
                const uint4 l1 = *reinterpret_cast<const uint4 *>(sb + p2 * 4 * G::ROW + 16 * kc_lo_swz(2 * lt + 1));
                const uint2 h = *reinterpret_cast<const uint2 *>(sb + (8 + p2) * G::ROW + 8 * lt);
                const unsigned lo[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
                double *acc = p2 ? acc1 : acc0;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const unsigned hb = ((k < 4 ? h.x : h.y) >> (8 * (k & 3))) & 0xffu;
                    const double kv = __hiloint2double((int)(0x43300000u | hb), (int)lo[k]) - F64_2P52;
                    acc[k] += f64_mac_term(v[k], kv, qq.x, qq.y);
                }
            }
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(skb + 2 * kswz(4 * lt + k, rin));
                const ulonglong2 y = *reinterpret_cast<const ulonglong2 *>(ska + 2 * kswz(4 * lt + k, rin));
                acc0[2 * k] += f64_mac_term(v[2 * k], u2d(x.x), qq.x, qq.y);
                acc0[2 * k + 1] += f64_mac_term(v[2 * k + 1], u2d(x.y), qq.x, qq.y);
                acc1[2 * k] += f64_mac_term(v[2 * k], u2d(y.x), qq.x, qq.y);
                acc1[2 * k + 1] += f64_mac_term(v[2 * k + 1], u2d(y.y), qq.x, qq.y);
            }
        }
        __syncwarp();  // key stage and row stage s consumed before they are refilled
        if (j + 1 < j1) issue_key(j + 1);
        cp_async_commit();
    }
    u64 o0[8], o1[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        o0[k] = f64_canon(acc0[k], qq.x, qq.y);
        o1[k] = f64_canon(acc1[k], qq.x, qq.y);
    }
    asm volatile("cp.async.wait_all;\n" ::);
    __syncwarp();
    const RowEx ex{sI[0][rin]};  // coalesced stores: element k at (k << (B2-3)) | lt
    if (a.rs_rows && t + 1 >= a.l && !a.part) {  // fused ModDown + rescale: z, then the INTT row phase
        if (t + 1 == a.l) {
            const u64 qi = __ldg(&tb.mod[prime].q);
            const ulonglong2 pm = __ldg(a.zrs + t);
            const u64 *b0 = limb_ptr(a.zbase, 2 * c, t, log_n) + roff + 8 * lt;
            const u64 *b1 = limb_ptr(a.zbase, 2 * c + 1, t, log_n) + roff + 8 * lt;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                o0[k] = addmod(shoup(b0[k], pm.x, pm.y, qi), o0[k], qi);
                o1[k] = addmod(shoup(b1[k], pm.x, pm.y, qi), o1[k], qi);
            }
        }
        const double2 *itwf = tb.ipsif + ((size_t)prime << log_n);  // ends in the coalesced layout
        inv_tile_f64<B2>(o0, ex, lt, B1, row, itwf);
        inv_tile_f64<B2>(o1, ex, lt, B1, row, itwf);
    } else {
        ex(o0, lt, 0, B2 - 3);
        ex(o1, lt, 0, B2 - 3);
    }
    u64 *e0 = a.part ? a.part + ((((size_t)blockIdx.y * a.cnt_run + c) * 2 * a.T + tl) << log_n) + roff
                     : a.ext + (((size_t)c * 2 * next + t) << log_n) + roff;
    u64 *e1 = e0 + ((size_t)(a.part ? a.T : next) << log_n);
    if (a.accum) {  // digit window after the first: add to the windows summed so far
        const u64 qa = __ldg(&tb.mod[prime].q);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            e0[(k << (B2 - 3)) | lt] = addmod(o0[k], e0[(k << (B2 - 3)) | lt], qa);
            e1[(k << (B2 - 3)) | lt] = addmod(o1[k], e1[(k << (B2 - 3)) | lt], qa);
        }
        return;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        e0[(k << (B2 - 3)) | lt] = o0[k];
        e1[(k << (B2 - 3)) | lt] = o1[k];
    }
}

// Integer-pipe counterpart of ks_mac_body_f64 (same shared-memory layout and pipeline: single
// key stage, cached row twiddles, the row stage as exchange buffer); Acc128 / Acc40 MACs.
template <int B2, class Acc, bool LAZY>
__device__ __forceinline__ void ks_mac_body_int(const MacArgs &a, const Tables &tb, u32 ngroups,
                                                u64 (*sI)[MacGeom<B2>::R][MacGeom<B2>::SROW],
                                                u64 (*sk)[2 * MacGeom<B2>::ROW], ulonglong2 *tws, u32 tile)
{
    using G = MacGeom<B2>;
    const u32 log_n = tb.log_n;
    const u32 B1 = log_n - B2;
    const u32 cr = tile >> (31 - __clz(ngroups)), grp = tile & (ngroups - 1);
    const u32 c = a.fT.div(cr), tl = cr - c * a.T;
    const u32 t = a.t0 + tl;
    const u32 ct = c * a.Ti + (t - a.t0i);
    const int rin = threadIdx.x / G::THR, lt = threadIdx.x % G::THR;
    const u32 row = grp * G::R + rin;
    const u32 prime = (t < a.l) ? t : a.sp;
    const u32 klimb = (t < a.l) ? t : a.Lk;
    const ulonglong2 *twf = tb.psi + ((size_t)prime << log_n);
    const ModC m = load_mod(tb.mod, prime);
    const size_t nn = (size_t)1 << log_n;
    const u32 roff = row << B2;
    const u64 *dp = limb_ptr(a.din, c, t < a.l ? t : 0, log_n);
    u64 *skb = sk[rin], *ska = skb + G::ROW;
    // Row-phase twiddles of this CTA's R rows, cached in shared memory once and reused by every
    // digit (they depend on the target and the rows only): stage s of row rin needs the 2^s
    // entries at 2^(B1+s) + row 2^s ...; the cache keeps them at R 2^s + rin 2^s ..., i.e. the
    // ntt.cuh index formula with k = log2 R and hi = rin.  (From L2 they were the kernel's top
    // long-scoreboard stall: ncu profiles/ncu_r1_v7_k_ks_mac.txt.)
    constexpr int LOGR = ilog2c(G::R);
    static_assert((1 << LOGR) == G::R, "rows per CTA is a power of two");
    {  // each warp fills its own rows' entries (so a __syncwarp publishes them)
        constexpr int RPW = 32 / G::THR;  // rows per warp
        const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
        for (int st = 0; st < B2; ++st) {
            const int cnt = RPW << st;
            const auto *src = twf + (1u << (B1 + st)) + ((size_t)(grp * G::R + w * RPW) << st);
            auto *dst = tws + (G::R << st) + ((w * RPW) << st);
            for (int e = lane; e < cnt; e += 32) cp_async16(dst + tw_cache_swz((u32)(((w * RPW) << st) + e), st) - ((w * RPW) << st), src + e);
        }
    }

    auto issue_row = [&](u32 j, int s) {
        u64 *d = sI[s][rin];
        if (j == t) {
            if (a.perm) {
#pragma unroll
                for (int i = 0; i < 8; ++i) cp_async8(d + dg_swz(8 * lt + i), dp + __ldg(a.perm + roff + 8 * lt + i));
            } else {
#pragma unroll
                for (int k = 0; k < G::CH; ++k) {
                    const int ch = lt + G::THR * k;
                    cp_async16(d + 2 * dg_cswz(ch), dp + roff + 2 * ch);
                }
            }
        } else {
            const u64 *ip = a.I + ((((size_t)ct * a.l) + j) << log_n) + roff;
#pragma unroll
            for (int k = 0; k < G::CH; ++k) {
                const int ch = lt + G::THR * k;
                cp_async16(d + 2 * ch, ip + 2 * ch);
            }
        }
    };
    auto issue_key = [&](u32 j) {
        const u64 *kb = a.key + ((size_t)(2 * j) * (a.Lk + 1) + klimb) * nn + roff;
        const u64 *ka = kb + (size_t)(a.Lk + 1) * nn;
#pragma unroll
        for (int k = 0; k < G::CH; ++k) {
            const int ch = lt + G::THR * k;
            cp_async16(skb + 2 * kswz(ch, rin), kb + 2 * ch);
            cp_async16(ska + 2 * kswz(ch, rin), ka + 2 * ch);
        }
    };

    Acc acc0[8], acc1[8];
    // commit groups, in order: row_0, key_0, then per digit j: row_{j+1}, key_{j+1}
    const u32 jwe = a.jw1 ? a.jw1 : a.l;
    const u32 j0 = a.jw0 + (a.part ? blockIdx.y * a.jper : 0), j1 = a.part ? min(jwe, j0 + a.jper) : jwe;
    issue_row(j0, 0);
    cp_async_commit();
    issue_key(j0);
    cp_async_commit();
    for (u32 j = j0; j < j1; ++j) {
        const int s = (j - j0) & 1;
        if (j + 1 < j1) issue_row(j + 1, s ^ 1);
        cp_async_commit();
        asm volatile("cp.async.wait_group 2;\n" ::);  // row_j landed (key_j, row_{j+1} may pend)
        __syncwarp();
        u64 v[8];
        if (j == t) {
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = sI[s][rin][dg_swz(8 * lt + k)];
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = sI[s][rin][(k << (B2 - 3)) | lt];
            // the row stage is free once loaded (refilled only next iteration): exchange buffer
            fwd_rounds_t<B2, 0, LAZY, RowEx, true>(v, RowEx{sI[s][rin]}, lt, LOGR, (u32)rin, tws, m.q);
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = LAZY ? reduce64(v[k], m.q, m.bar) : csub(csub(v[k], 2 * m.q), m.q);
        }
        cp_async_wait1();  // key_j landed (row_{j+1} may pend)
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(skb + 2 * kswz(4 * lt + k, rin));
            const ulonglong2 y = *reinterpret_cast<const ulonglong2 *>(ska + 2 * kswz(4 * lt + k, rin));
            acc0[2 * k].mac(v[2 * k], x.x);
            acc0[2 * k + 1].mac(v[2 * k + 1], x.y);
            acc1[2 * k].mac(v[2 * k], y.x);
            acc1[2 * k + 1].mac(v[2 * k + 1], y.y);
        }
        __syncwarp();  // key stage and row stage s consumed before they are refilled
        if (j + 1 < j1) issue_key(j + 1);
        cp_async_commit();
    }
    u64 o0[8], o1[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        o0[k] = acc0[k].reduce(m);
        o1[k] = acc1[k].reduce(m);
    }
    asm volatile("cp.async.wait_all;\n" ::);
    __syncwarp();
    const RowEx ex{sI[0][rin]};  // coalesced stores: element k at (k << (B2-3)) | lt
    if (a.pinv_rows && t == a.l && !a.part) {  // inverse row phase instead of the plain exchange:
        const ulonglong2 *itw = tb.ipsi + ((size_t)prime << log_n);  // it ends in the same layout
        inv_rounds<B2, 0>(o0, ex, lt, B1, row, itw, m.q, 0, tb.ipsif + ((size_t)prime << log_n), false);
        inv_rounds<B2, 0>(o1, ex, lt, B1, row, itw, m.q, 0, tb.ipsif + ((size_t)prime << log_n), false);
    } else {
        ex(o0, lt, 0, B2 - 3);
        ex(o1, lt, 0, B2 - 3);
    }
    u64 *e0 = a.part ? a.part + ((((size_t)blockIdx.y * a.cnt_run + c) * 2 * a.T + tl) << log_n) + roff
                     : a.ext + (((size_t)c * 2 * (a.l + 1) + t) << log_n) + roff;
    u64 *e1 = e0 + ((size_t)(a.part ? a.T : a.l + 1) << log_n);
    if (a.accum) {  // digit window after the first: add to the windows summed so far
        const u64 qa = __ldg(&tb.mod[(t < a.l) ? t : a.sp].q);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            e0[(k << (B2 - 3)) | lt] = addmod(o0[k], e0[(k << (B2 - 3)) | lt], qa);
            e1[(k << (B2 - 3)) | lt] = addmod(o1[k], e1[(k << (B2 - 3)) | lt], qa);
        }
        return;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        e0[(k << (B2 - 3)) | lt] = o0[k];
        e1[(k << (B2 - 3)) | lt] = o1[k];
    }
}

// One code path per kernel (the digit loop is ~1.4k instructions; two paths in flight
// thrash the instruction cache): the host launches each run of targets of one class
// separately.  CLS 2: Acc40 (q < 2^40, long digit loops: fewer IMAD.WIDE per MAC, ~40 more
// registers); CLS 1: Acc128 + lazy NTT (q < 2^48); CLS 0: Acc128 + Harvey NTT;
// CLS 5: FP64 NTT + FP64 inner product (ks_mac_body_f64), every FP64-mode target (its ModUp
// slabs hold lazy doubles); CLS 6/7: the integer classes on the CLS 5 pipeline.
#ifndef KSMAC5_BLOCKS
#define KSMAC5_BLOCKS 8
#endif
template <int B2, int CLS>
__global__ void __launch_bounds__(64, CLS == 2 ? 6 : CLS == 5 ? KSMAC5_BLOCKS : 8) k_ks_mac(MacArgs a, Tables tb, u32 ngroups)
{
    using G = MacGeom<B2>;
    if constexpr (CLS == 5) {
        __shared__ __align__(16) u64 sI[2][G::R][G::SROW];
        __shared__ __align__(16) u64 sk[G::R][2 * G::ROW];
        __shared__ __align__(16) double2 tws[G::R << B2];
        ks_mac_body_f64<B2>(a, tb, ngroups, sI, sk, tws, blockIdx.x);
        return;
    }
    if constexpr (CLS == 6 || CLS == 7) {  // integer classes on the CLS 5 pipeline (lazy / Harvey NTT)
        __shared__ __align__(16) u64 sI[2][G::R][G::SROW];
        __shared__ __align__(16) u64 sk[G::R][2 * G::ROW];
        __shared__ __align__(16) ulonglong2 tws[G::R << B2];
        ks_mac_body_int<B2, Acc128, CLS == 6>(a, tb, ngroups, sI, sk, tws, blockIdx.x);
        return;
    }
    __shared__ __align__(16) u64 buf[2][G::R][G::STAGE];
    __shared__ u64 sx[G::R * G::SROW];
    if constexpr (CLS == 2)
        ks_mac_body<B2, Acc40, true>(a, tb, ngroups, buf, sx);
    else
        ks_mac_body<B2, Acc128, CLS == 1>(a, tb, ngroups, buf, sx);
}

// ------------------------------------------------------------------------------------
// Inverse: row phase first (stages logN-1..B1), then column phase (B1-1..0) with N^{-1}.
// ------------------------------------------------------------------------------------
template <int B2>
__global__ void __launch_bounds__(128) k_inv_rows(TaskPlainCol task, const u32 *perm, Tables tb, u32 ngroups)
{
    using G = RowGeom<B2>;
    __shared__ u64 sm[G::R * G::SROW];
    const u32 log_n = tb.log_n;
    const u32 B1 = log_n - B2;
    const u32 r = blockIdx.x >> (31 - __clz(ngroups)), grp = blockIdx.x & (ngroups - 1);
    const int rin = threadIdx.x / G::THR, lt = threadIdx.x % G::THR;
    const u32 row = grp * G::R + rin;
    const u64 *src;
    u64 *dst;
    u32 prime, sprime;
    task.get(r, src, dst, prime, sprime);
    const ModC m = load_mod(tb.mod, prime);
    const ulonglong2 *itw = tb.ipsi + ((size_t)prime << log_n);
    const bool f64 = use_f64(tb, m.q);
    const u32 roff = row << B2;
    u64 v[8];  // coalesced loads (element k at (k << (B2-3)) | lt), then to the first GS layout
    if (perm) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = src[__ldg(perm + roff + ((k << (B2 - 3)) | lt))];
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = src[roff + ((k << (B2 - 3)) | lt)];
    }
    const RowEx ex{sm + rin * G::SROW};
    ex(v, lt, B2 - 3, 0);
    inv_rounds<B2, 0>(v, ex, lt, B1, row, itw, m.q, 0, tb.ipsif + ((size_t)prime << log_n), f64);
    u64 *drow = dst + ((size_t)row << B2);
#pragma unroll
    for (int i = 0; i < 8; ++i) drow[(i << (B2 - 3)) | lt] = v[i];
}

// HMULT tensor product fused with the first half of the relinearisation digits' INTT: a CTA
// owns R rows of limb i of ciphertext c, computes (d0, d1, d2) = (a0 b0, a0 b1 + a1 b0, a1 b1)
// mod q_i for its row elements (d0, d1 stored as k_elem<FTensor> does), stores d2 in NTT form (the
// key switch's diagonal digits read it) and runs the inverse row phase on d2 straight from
// registers into dr -- the row-phase launch of the digits' INTT and its HBM round trip vanish.
struct TensorRows {
    PolyMap a, b, out, d2, dr;
    u32 l;
    FDiv fl{};
};
template <int B2>
__global__ void __launch_bounds__(128) k_tensor_inv_rows(TensorRows t, Tables tb, u32 ngroups)
{
    using G = RowGeom<B2>;
    __shared__ u64 sm[G::R * G::SROW];
    const u32 log_n = tb.log_n;
    const u32 B1 = log_n - B2;
    const u32 r = blockIdx.x >> (31 - __clz(ngroups)), grp = blockIdx.x & (ngroups - 1);
    const u32 c = t.fl.div(r), i = r - c * t.l;
    const int rin = threadIdx.x / G::THR, lt = threadIdx.x % G::THR;
    const u32 row = grp * G::R + rin;
    const ModC m = load_mod(tb.mod, i);
    const bool f64 = use_f64(tb, m.q);
    const u32 roff = row << B2;
    const u64 *a0 = limb_ptr(t.a, 2 * c, i, log_n) + roff, *a1 = limb_ptr(t.a, 2 * c + 1, i, log_n) + roff;
    const u64 *b0 = limb_ptr(t.b, 2 * c, i, log_n) + roff, *b1 = limb_ptr(t.b, 2 * c + 1, i, log_n) + roff;
    u64 *o0 = limb_ptr_w(t.out, 2 * c, i, log_n) + roff, *o1 = limb_ptr_w(t.out, 2 * c + 1, i, log_n) + roff;
    u64 *dn = limb_ptr_w(t.d2, c, i, log_n) + roff;
    u64 v[8];
    // every operand of the thread is loaded before the first store: out may alias a or b (in-place
    // HMULT), so the compiler would otherwise keep each element's loads behind the previous
    // element's stores and serialise eight HBM round trips (ncu: 50 % of DRAM peak)
    u64 X0[8], X1[8], Y0[8], Y1[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int e = (k << (B2 - 3)) | lt;
        X0[k] = a0[e];
        X1[k] = a1[e];
        Y0[k] = b0[e];
        Y1[k] = b1[e];
    }
    if (f64) {  // FP64 pipe: exact two-product terms (canonical inputs < q < 2^42), as FTensor
        const double2 qq = __ldg(tb.psif + ((size_t)i << log_n));
        auto mm = [&](u64 x, u64 y) { return f64_mac_term(u2d(x), u2d(y), qq.x, qq.y); };
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int e = (k << (B2 - 3)) | lt;
            const u64 x0 = X0[k], x1 = X1[k], y0 = Y0[k], y1 = Y1[k];
            o0[e] = f64_canon(mm(x0, y0), qq.x, qq.y);
            o1[e] = f64_canon(mm(x0, y1) + mm(x1, y0), qq.x, qq.y);
            v[k] = f64_canon(mm(x1, y1), qq.x, qq.y);
            dn[e] = v[k];
        }
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int e = (k << (B2 - 3)) | lt;
            const u64 x0 = X0[k], x1 = X1[k], y0 = Y0[k], y1 = Y1[k];
            o0[e] = mulmod(x0, y0, m);
            u64 lo = 0, hi = 0;
            mac128(lo, hi, x0, y1);
            mac128(lo, hi, x1, y0);
            o1[e] = reduce128(lo, hi, m);
            v[k] = mulmod(x1, y1, m);
            dn[e] = v[k];
        }
    }
    const RowEx ex{sm + rin * G::SROW};
    ex(v, lt, B2 - 3, 0);
    inv_rounds<B2, 0>(v, ex, lt, B1, row, tb.ipsi + ((size_t)i << log_n), m.q, 0, tb.ipsif + ((size_t)i << log_n), f64);
    u64 *drow = limb_ptr_w(t.dr, c, i, log_n) + roff;
#pragma unroll
    for (int k = 0; k < 8; ++k) drow[(k << (B2 - 3)) | lt] = v[k];
}

template <int B1, int B2>
__global__ void __launch_bounds__(COLS *(1 << B1) / 8) k_inv_cols(TaskPlainCol task, Tables tb, u32 ngroups)
{
    __shared__ u64 sm[(1 << B1) * COLS];
    constexpr u32 log_n = B1 + B2, n2 = 1u << B2;
    const u32 r = blockIdx.x >> (31 - __clz(ngroups)), grp = blockIdx.x & (ngroups - 1);
    const int col = threadIdx.x % COLS, lt = threadIdx.x / COLS;
    const u64 *src;
    u64 *dst;
    u32 prime, sprime;
    task.get(r, src, dst, prime, sprime);
    const ModC m = load_mod(tb.mod, prime);
    const ulonglong2 *itw = tb.ipsi + ((size_t)prime << log_n);
    const ulonglong2 ni = __ldg(tb.ninv + prime);
    const u32 c = grp * COLS + col;
    u64 v[8];
    const u64 *lp0 = dst + (size_t)(lt << 3) * n2 + c;  // element i at lidx(lt, i, 0) = 8 lt + i
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = lp0[(size_t)i * n2];
    inv_rounds<B1, 0>(v, ColEx<COLS>{sm, col}, lt, 0, 0u, itw, m.q, (int)(log_n - B1),
                      tb.ipsif + ((size_t)prime << log_n), use_f64(tb, m.q));
    u64 *sp0 = dst + (size_t)lt * n2 + c;  // element i at ((i << (B1-3)) | lt) * n2 + c
#pragma unroll
    for (int i = 0; i < 8; ++i) sp0[(size_t)i << (B1 - 3 + B2)] = shoup(v[i], ni.x, ni.y, m.q);
}

// ------------------------------------------------------------------------------------
// Key-switch digits straight into ModUp: the inverse column phase of digit j (of a CTA's 16
// columns) leaves the coefficient-form digit D_j in the exact register layout the forward
// column phase starts from ((i << (B1-3)) | lt), so the same CTA continues with the forward
// column phase of D_j under every target t != j and stores the ModUp slabs I[c][t][j].
// D never goes to memory (the two-kernel path wrote it and re-read it once per target).
// ------------------------------------------------------------------------------------
struct InvModUpArgs {
    TaskPlainCol inv;  // row-phase output of the digits' INTT, [cnt][l][N] (limb j = digit j)
    u64 *I;            // [cnt][T][l][N] ModUp column-phase slabs
    u32 l, t0, T, sp;
};

template <int B1, int B2>
__global__ void __launch_bounds__(COLS *(1 << B1) / 8) k_inv_cols_modup(InvModUpArgs a, Tables tb, u32 ngroups)
{
    __shared__ u64 sm[(1 << B1) * COLS];
    constexpr u32 log_n = B1 + B2, n2 = 1u << B2;
    const u32 r = blockIdx.x >> (31 - __clz(ngroups)), grp = blockIdx.x & (ngroups - 1);
    const int col = threadIdx.x % COLS, lt = threadIdx.x / COLS;
    const u64 *src;
    u64 *dst;
    u32 jprime, sprime;
    a.inv.get(r, src, dst, jprime, sprime);  // r = c * l + j, prime of limb j = j
    const u32 c = r / a.l, j = r - c * a.l;
    const ModC mj = load_mod(tb.mod, jprime);
    const ulonglong2 ni = __ldg(tb.ninv + jprime);
    const u32 cc = grp * COLS + col;
    u64 d[8];
    {
        const u64 *lp0 = dst + (size_t)(lt << 3) * n2 + cc;  // row-phase output, in place in dst
#pragma unroll
        for (int i = 0; i < 8; ++i) d[i] = lp0[(size_t)i * n2];
        inv_rounds<B1, 0>(d, ColEx<COLS>{sm, col}, lt, 0, 0u, tb.ipsi + ((size_t)jprime << log_n), mj.q, (int)B2,
                          tb.ipsif + ((size_t)jprime << log_n), use_f64(tb, mj.q));
#pragma unroll
        for (int i = 0; i < 8; ++i) d[i] = shoup(d[i], ni.x, ni.y, mj.q);  // canonical D_j
    }
    for (u32 tl = 0; tl < a.T; ++tl) {
        const u32 t = a.t0 + tl;
        if (t == j) continue;  // the diagonal digit reuses d's own NTT-form limb (ks_mac)
        const u32 prime = (t < a.l) ? t : a.sp;
        const ModC m = load_mod(tb.mod, prime);
        const bool f64 = use_f64(tb, m.q);
        const bool red = f64 ? !use_f64(tb, mj.q) : mj.q > m.q;  // as k_fwd_cols (TaskModUpCol)
        u64 v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = red ? reduce64(d[i], m.q, m.bar) : d[i];
        if (f64)  // FP64-mode target: the slab holds lazy doubles (k_ks_mac CLS 5 reads them as such)
            fwd_tile_f64_raw<B1>(v, ColEx<COLS>{sm, col}, lt, 0, 0u, tb.psif + ((size_t)prime << log_n));
        else
            fwd_rounds<B1, 0>(v, ColEx<COLS>{sm, col}, lt, 0, 0u, tb.psi + ((size_t)prime << log_n), m.q,
                              tb.psif + ((size_t)prime << log_n), f64);
        if (!f64 && lazy_wide<B1>(m.q)) {
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = reduce64(v[i], m.q, m.bar);
        }
        u64 *dp0 = a.I + ((((size_t)c * a.T + tl) * a.l + j) << log_n) + (size_t)(lt << 3) * n2 + cc;
#pragma unroll
        for (int i = 0; i < 8; ++i) dp0[(size_t)i * n2] = v[i];
    }
}

// ModDown / rescale broadcast, fused the same way: the inverse column phase of the source limb
// (the special-prime accumulator, or the ciphertext's last limb) leaves its coefficient form
// in the forward column layout, and the CTA runs the broadcast's forward column phase under
// every target q_t straight from registers into S[p][t - toff].
struct InvBcastArgs {
    TaskPlainCol inv;  // one source limb per polynomial (ls.n = 1): row-phase output in inv.dst
    u64 *S;            // [npolys][nt][N]
    u32 nt, toff;
};

template <int B1, int B2>
__global__ void __launch_bounds__(COLS *(1 << B1) / 8) k_inv_cols_bcast(InvBcastArgs a, Tables tb, u32 ngroups)
{
    __shared__ u64 sm[(1 << B1) * COLS];
    constexpr u32 log_n = B1 + B2, n2 = 1u << B2;
    const u32 r = blockIdx.x >> (31 - __clz(ngroups)), grp = blockIdx.x & (ngroups - 1);  // r = polynomial
    const int col = threadIdx.x % COLS, lt = threadIdx.x / COLS;
    const u64 *src;
    u64 *dst;
    u32 sprime, dummy;
    a.inv.get(r, src, dst, sprime, dummy);
    const ModC ms = load_mod(tb.mod, sprime);
    const ulonglong2 ni = __ldg(tb.ninv + sprime);
    const u32 cc = grp * COLS + col;
    u64 x[8];
    {
        const u64 *lp0 = dst + (size_t)(lt << 3) * n2 + cc;
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = lp0[(size_t)i * n2];
        inv_rounds<B1, 0>(x, ColEx<COLS>{sm, col}, lt, 0, 0u, tb.ipsi + ((size_t)sprime << log_n), ms.q, (int)B2,
                          tb.ipsif + ((size_t)sprime << log_n), use_f64(tb, ms.q));
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = shoup(x[i], ni.x, ni.y, ms.q);
    }
    for (u32 i = 0; i < a.nt; ++i) {
        const u32 t = a.toff + i;
        const ModC m = load_mod(tb.mod, t);
        const bool f64 = use_f64(tb, m.q);
        const bool red = f64 ? !use_f64(tb, ms.q) : ms.q > m.q;  // as k_fwd_cols (TaskBcastCol)
        u64 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = red ? reduce64(x[k], m.q, m.bar) : x[k];
        fwd_rounds<B1, 0>(v, ColEx<COLS>{sm, col}, lt, 0, 0u, tb.psi + ((size_t)t << log_n), m.q,
                          tb.psif + ((size_t)t << log_n), f64);
        if (!f64 && lazy_wide<B1>(m.q)) {
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = reduce64(v[k], m.q, m.bar);
        }
        u64 *dp0 = a.S + (((size_t)r * a.nt + i) << log_n) + (size_t)(lt << 3) * n2 + cc;
#pragma unroll
        for (int k = 0; k < 8; ++k) dp0[(size_t)k * n2] = v[k];
    }
}

// ------------------------------------------------------------------------------------
// Elementwise kernels: 2 coefficients per thread, grid-stride.
// ------------------------------------------------------------------------------------
template <class F>
__global__ void __launch_bounds__(256) k_elem(F f, u32 npolys, u32 l, u32 log_n, const ModC *mods, FDiv fl)
{
    const size_t total = ((size_t)npolys * l) << (log_n - 1);
    for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
        const size_t e = t << 1;
        const u32 idx = (u32)(e & ((1u << log_n) - 1));
        const u32 pl = (u32)(e >> log_n);  // polynomial-limb index (< 2^32)
        const u32 p = fl.div(pl), i = pl - p * l;
        f(p, i, idx, mods[i], log_n);
    }
}

struct FAddSub {
    static constexpr const char *NAME = "elem_addsub";
    static constexpr double MULS = 0, WORDS = 3;
    PolyMap a, b, out;
    int op;
    __device__ void operator()(u32 p, u32 i, u32 idx, const ModC &m, u32 log_n) const
    {
        const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(limb_ptr(a, p, i, log_n) + idx);
        const ulonglong2 y = *reinterpret_cast<const ulonglong2 *>(limb_ptr(b, p, i, log_n) + idx);
        ulonglong2 o;
        if (op == EL_ADD) {
            o.x = addmod(x.x, y.x, m.q);
            o.y = addmod(x.y, y.y, m.q);
        } else {
            o.x = submod(x.x, y.x, m.q);
            o.y = submod(x.y, y.y, m.q);
        }
        *reinterpret_cast<ulonglong2 *>(limb_ptr_w(out, p, i, log_n) + idx) = o;
    }
};

struct FMulPoly {
    static constexpr const char *NAME = "elem_mulpoly";
    static constexpr double MULS = 1, WORDS = 3;
    PolyMap a, b, out;
    u32 b_div, b_mod;
    __device__ void operator()(u32 p, u32 i, u32 idx, const ModC &m, u32 log_n) const
    {
        const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(limb_ptr(a, p, i, log_n) + idx);
        const u32 pb = b_mod ? (p / b_div) % b_mod : p / b_div;
        const ulonglong2 y = *reinterpret_cast<const ulonglong2 *>(limb_ptr(b, pb, i, log_n) + idx);
        *reinterpret_cast<ulonglong2 *>(limb_ptr_w(out, p, i, log_n) + idx) =
            make_ulonglong2(mulmod(x.x, y.x, m), mulmod(x.y, y.y, m));
    }
};

struct FAddPlain {  // over ciphertexts x 2 polys: c0 += pt
    static constexpr const char *NAME = "elem_addplain";
    static constexpr double MULS = 0, WORDS = 3;
    PolyMap ct, pt, out;
    u32 bcast;
    __device__ void operator()(u32 p, u32 i, u32 idx, const ModC &m, u32 log_n) const
    {
        ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(limb_ptr(ct, p, i, log_n) + idx);
        if ((p & 1) == 0) {
            const u32 pp = bcast ? 0 : p / 2;
            const ulonglong2 y = *reinterpret_cast<const ulonglong2 *>(limb_ptr(pt, pp, i, log_n) + idx);
            x.x = addmod(x.x, y.x, m.q);
            x.y = addmod(x.y, y.y, m.q);
        }
        *reinterpret_cast<ulonglong2 *>(limb_ptr_w(out, p, i, log_n) + idx) = x;
    }
};

struct FMulScalar {
    static constexpr const char *NAME = "elem_mulscalar";
    static constexpr double MULS = 1, WORDS = 2;
    PolyMap a, out;
    const ulonglong2 *c;
    __device__ void operator()(u32 p, u32 i, u32 idx, const ModC &m, u32 log_n) const
    {
        const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(limb_ptr(a, p, i, log_n) + idx);
        const ulonglong2 w = __ldg(c + i);
        *reinterpret_cast<ulonglong2 *>(limb_ptr_w(out, p, i, log_n) + idx) =
            make_ulonglong2(shoup(x.x, w.x, w.y, m.q), shoup(x.y, w.x, w.y, m.q));
    }
};

struct FAddScalarC0 {
    static constexpr const char *NAME = "elem_addscalar";
    static constexpr double MULS = 0, WORDS = 2;
    PolyMap ct, out;
    const u64 *c;
    __device__ void operator()(u32 p, u32 i, u32 idx, const ModC &m, u32 log_n) const
    {
        ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(limb_ptr(ct, p, i, log_n) + idx);
        if ((p & 1) == 0) {
            const u64 w = __ldg(c + i);
            x.x = addmod(x.x, w, m.q);
            x.y = addmod(x.y, w, m.q);
        }
        *reinterpret_cast<ulonglong2 *>(limb_ptr_w(out, p, i, log_n) + idx) = x;
    }
};

struct FTensor {  // p = output ciphertext; inputs paired as a[(p / adiv) % amod], b[(p / bdiv) % bmod]
    static constexpr const char *NAME = "elem_tensor";
    static constexpr double MULS = 4, WORDS = 7;
    PolyMap a, b, out, d2;
    u32 adiv, amod, bdiv, bmod;  // amod/bmod = 0: no wrap
    const double2 *psif = nullptr;  // FP64-mode primes: (q, 1/q) at psif[prime << log_n] (else null)
    u64 f64_qmax = 0;
    __device__ void operator()(u32 p, u32 i, u32 idx, const ModC &m, u32 log_n) const
    {
        const u32 qa = adiv == 1 ? p : p / adiv, qb = bdiv == 1 ? p : p / bdiv;  // (1: the plain HMULT)
        const u32 pa = amod ? qa % amod : qa, pb = bmod ? qb % bmod : qb;
        const ulonglong2 a0 = *reinterpret_cast<const ulonglong2 *>(limb_ptr(a, 2 * pa, i, log_n) + idx);
        const ulonglong2 a1 = *reinterpret_cast<const ulonglong2 *>(limb_ptr(a, 2 * pa + 1, i, log_n) + idx);
        const ulonglong2 b0 = *reinterpret_cast<const ulonglong2 *>(limb_ptr(b, 2 * pb, i, log_n) + idx);
        const ulonglong2 b1 = *reinterpret_cast<const ulonglong2 *>(limb_ptr(b, 2 * pb + 1, i, log_n) + idx);
        ulonglong2 d0, d1, dd;
        if (m.q < f64_qmax) {  // FP64 pipe: exact two-product terms (canonical inputs < q < 2^42)
            const double2 qq = __ldg(psif + ((size_t)i << log_n));
            auto mm = [&](u64 x, u64 y) { return f64_mac_term(u2d(x), u2d(y), qq.x, qq.y); };
            d0 = make_ulonglong2(f64_canon(mm(a0.x, b0.x), qq.x, qq.y), f64_canon(mm(a0.y, b0.y), qq.x, qq.y));
            d1 = make_ulonglong2(f64_canon(mm(a0.x, b1.x) + mm(a1.x, b0.x), qq.x, qq.y),
                                 f64_canon(mm(a0.y, b1.y) + mm(a1.y, b0.y), qq.x, qq.y));
            dd = make_ulonglong2(f64_canon(mm(a1.x, b1.x), qq.x, qq.y), f64_canon(mm(a1.y, b1.y), qq.x, qq.y));
        } else {
            d0.x = mulmod(a0.x, b0.x, m);
            d0.y = mulmod(a0.y, b0.y, m);
            {
                u64 lo = 0, hi = 0;
                mac128(lo, hi, a0.x, b1.x);
                mac128(lo, hi, a1.x, b0.x);
                d1.x = reduce128(lo, hi, m);
                lo = hi = 0;
                mac128(lo, hi, a0.y, b1.y);
                mac128(lo, hi, a1.y, b0.y);
                d1.y = reduce128(lo, hi, m);
            }
            dd.x = mulmod(a1.x, b1.x, m);
            dd.y = mulmod(a1.y, b1.y, m);
        }
        *reinterpret_cast<ulonglong2 *>(limb_ptr_w(out, 2 * p, i, log_n) + idx) = d0;
        *reinterpret_cast<ulonglong2 *>(limb_ptr_w(out, 2 * p + 1, i, log_n) + idx) = d1;
        *reinterpret_cast<ulonglong2 *>(limb_ptr_w(d2, p, i, log_n) + idx) = dd;
    }
};

struct FFromSigned {
    static constexpr const char *NAME = "elem_fromsigned";
    static constexpr double MULS = 0, WORDS = 2;
    const int64_t *e;
    PolyMap out;
    __device__ void operator()(u32 p, u32 i, u32 idx, const ModC &m, u32 log_n) const
    {
        const int64_t *src = e + ((size_t)p << log_n) + idx;
        u64 o[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int64_t x = src[k];
            const u64 ax = (u64)(x < 0 ? -x : x);
            const u64 rr = reduce64(ax, m.q, m.bar);
            o[k] = (x < 0 && rr) ? m.q - rr : rr;
        }
        *reinterpret_cast<ulonglong2 *>(limb_ptr_w(out, p, i, log_n) + idx) = make_ulonglong2(o[0], o[1]);
    }
};

struct FCopy {
    static constexpr const char *NAME = "elem_copy";
    static constexpr double MULS = 0, WORDS = 2;
    PolyMap src, dst;
    __device__ void operator()(u32 p, u32 i, u32 idx, const ModC &, u32 log_n) const
    {
        *reinterpret_cast<ulonglong2 *>(limb_ptr_w(dst, p, i, log_n) + idx) =
            *reinterpret_cast<const ulonglong2 *>(limb_ptr(src, p, i, log_n) + idx);
    }
};

struct FPermute {
    static constexpr const char *NAME = "elem_permute";
    static constexpr double MULS = 0, WORDS = 2;
    PolyMap src, dst;
    const u32 *perm;
    __device__ void operator()(u32 p, u32 i, u32 idx, const ModC &, u32 log_n) const
    {
        const u64 *s = limb_ptr(src, p, i, log_n);
        *reinterpret_cast<ulonglong2 *>(limb_ptr_w(dst, p, i, log_n) + idx) =
            make_ulonglong2(s[__ldg(perm + idx)], s[__ldg(perm + idx + 1)]);
    }
};

struct FMulAdd {  // out = (+/-) a*s + b
    static constexpr const char *NAME = "elem_muladd";
    static constexpr double MULS = 1, WORDS = 4;
    PolyMap a, s, b, out;
    u32 s_bcast;
    int neg;
    __device__ void operator()(u32 p, u32 i, u32 idx, const ModC &m, u32 log_n) const
    {
        const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(limb_ptr(a, p, i, log_n) + idx);
        const ulonglong2 y = *reinterpret_cast<const ulonglong2 *>(limb_ptr(s, s_bcast ? 0 : p, i, log_n) + idx);
        const ulonglong2 z = *reinterpret_cast<const ulonglong2 *>(limb_ptr(b, p, i, log_n) + idx);
        u64 t0 = mulmod(x.x, y.x, m), t1 = mulmod(x.y, y.y, m);
        ulonglong2 o;
        o.x = neg ? submod(z.x, t0, m.q) : addmod(z.x, t0, m.q);
        o.y = neg ? submod(z.y, t1, m.q) : addmod(z.y, t1, m.q);
        *reinterpret_cast<ulonglong2 *>(limb_ptr_w(out, p, i, log_n) + idx) = o;
    }
};

struct FKeygenB {  // p = digit j, i = limb in ext basis {q_0..q_{L-1}, p_0..p_{K-1}}
    static constexpr const char *NAME = "elem_keygen";
    static constexpr double MULS = 2, WORDS = 6;
    const u64 *a, *e, *s, *sfrom, *pmod;
    u64 *key;
    u32 Lk, K, alpha;
    __device__ void operator()(u32 j, u32 i, u32 idx, const ModC &m, u32 log_n) const
    {
        const size_t n = (size_t)1 << log_n, LK = Lk + K;
        const size_t ai = ((size_t)j * LK + i) * n + idx;
        const bool own = i < Lk && i / alpha == j;  // limb i belongs to digit j (A9 / f2)
        u64 o[2], aa[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            aa[k] = a[ai + k];
            u64 v = submod(e[ai + k], mulmod(aa[k], s[i * n + idx + k], m), m.q);
            if (own) v = addmod(v, mulmod(__ldg(pmod + i), sfrom[i * n + idx + k], m), m.q);
            o[k] = v;
        }
        const size_t kb = ((size_t)(2 * j) * LK + i) * n + idx;
        const size_t ka = ((size_t)(2 * j + 1) * LK + i) * n + idx;
        *reinterpret_cast<ulonglong2 *>(key + kb) = make_ulonglong2(o[0], o[1]);
        *reinterpret_cast<ulonglong2 *>(key + ka) = make_ulonglong2(aa[0], aa[1]);
    }
};

struct FModAddGathered {
    static constexpr const char *NAME = "elem_modadd_gathered";
    static constexpr double MULS = 0, WORDS = 3;
    const u64 *g;
    size_t stride;
    u32 R;
    PolyMap out;
    __device__ void operator()(u32 p, u32 i, u32 idx, const ModC &m, u32 log_n) const
    {
        const size_t o = (((size_t)p * out.cap + i) << log_n) + idx;
        u64 s0 = 0, s1 = 0;
        for (u32 r = 0; r < R; ++r) {
            const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(g + r * stride + o);
            s0 = addmod(s0, x.x, m.q);
            s1 = addmod(s1, x.y, m.q);
        }
        *reinterpret_cast<ulonglong2 *>(out.base + o) = make_ulonglong2(s0, s1);
    }
};

// out ciphertext q, poly k = sum_{r < R} g[ct r*rs + q*qs][poly k]  (reductions over a batch axis)
struct FSumStrided {
    static constexpr const char *NAME = "elem_sum";
    static constexpr double MULS = 0, WORDS = 3;
    PolyMap g, out;
    u32 R, rs, qs, np;
    __device__ void operator()(u32 p, u32 i, u32 idx, const ModC &m, u32 log_n) const
    {
        const u32 q = p / np, kk = p % np;
        u64 s0 = 0, s1 = 0;
        for (u32 r = 0; r < R; ++r) {
            const ulonglong2 x =
                *reinterpret_cast<const ulonglong2 *>(limb_ptr(g, (r * rs + q * qs) * np + kk, i, log_n) + idx);
            s0 = addmod(s0, x.x, m.q);
            s1 = addmod(s1, x.y, m.q);
        }
        *reinterpret_cast<ulonglong2 *>(limb_ptr_w(out, p, i, log_n) + idx) = make_ulonglong2(s0, s1);
    }
};

template <class F>
void run_elem(const Launch &L, const F &f, u32 npolys, u32 l)
{
    if (npolys == 0 || l == 0) return;
    const size_t total = ((size_t)npolys * l) << (L.tb->log_n - 1);
    size_t blocks = (total + 255) / 256;
    const size_t cap = (size_t)L.n_sm * 16;  // 16 resident 256-thread CTAs per SM worth of grid-stride work
    if (blocks > cap) blocks = cap;
    const double elems = (double)npolys * l * (1u << L.tb->log_n);
    KLAUNCH(L, F::NAME, (Work{0, elems * F::MULS, elems * 8.0 * F::WORDS}), (k_elem<F><<<(unsigned)blocks, 256, 0, L.st>>>(f, npolys, l, L.tb->log_n, L.tb->mod, make_fdiv(l))));
}

// ---- work accounting: which butterflies run on the FP64 pipe ---------------------------
bool f64_prime(const Launch &L, u32 prime) { return L.hprimes[prime] < L.tb->f64_qmax; }
double f64_share(const Launch &L, const LimbSet &ls)
{
    u32 k = 0;
    for (u32 i = 0; i < ls.n; ++i) k += f64_prime(L, i < ls.lq ? ls.qoff + i : ls.sp + (i - ls.lq)) ? 1 : 0;
    return ls.n ? (double)k / ls.n : 0.0;
}
double f64_share_range(const Launch &L, u32 p0, u32 n)
{
    u32 k = 0;
    for (u32 i = 0; i < n; ++i) k += f64_prime(L, p0 + i) ? 1 : 0;
    return n ? (double)k / n : 0.0;
}
Work nttw(double bfly, double f, double mac, double bytes) { return Work{bfly * (1 - f), mac, bytes, bfly * f}; }

// ---- NTT dispatch over log N ------------------------------------------------------
template <int B1, int B2>
void ntt_fwd_impl(const Launch &L, const TaskPlainCol &t, u32 nlimbs)
{
    const u32 log_n = L.tb->log_n;
    const u32 g1 = (1u << B2) / COLS;
    const double nh = (double)nlimbs * (1u << (B1 + B2 - 1)), nb = (double)nlimbs * (8u << (B1 + B2));
    const double f = f64_share(L, t.ls);
    TaskPlainCol t2 = t;
    t2.src = t.dst;  // row phase is in place on dst
    if (f == 1.0 && B1 >= 6) {  // every limb FP64-mode: radix-16 columns, the rows continue from lazy doubles
        KLAUNCH(L, "ntt_fwd_cols", nttw(nh * B1, f, 0, 2 * nb),
                (k_fwd_cols_r16<(B1 >= 6 ? B1 : 6), B2, TaskPlainCol><<<nlimbs * g1, 1 << B1, 0, L.st>>>(t, *L.tb, g1)));
        t2.raw = 1;
    } else {
        KLAUNCH(L, "ntt_fwd_cols", nttw(nh * B1, f, 0, 2 * nb), (k_fwd_cols<B1, B2, TaskPlainCol><<<nlimbs * g1, COLS * (1 << B1) / 8, 0, L.st>>>(t, *L.tb, g1)));
    }
    const u32 g2 = (1u << B1) / RowGeom<B2>::R;
    KLAUNCH(L, "ntt_fwd_rows", nttw(nh * B2, f, 0, 2 * nb), (k_fwd_rows_store<B2, TaskPlainCol><<<nlimbs * g2, 128, 0, L.st>>>(t2, *L.tb, g2)));
    (void)log_n;
}

template <int B1, int B2>
void ntt_inv_impl(const Launch &L, const TaskPlainCol &t, u32 nlimbs, const u32 *perm)
{
    const u32 g2 = (1u << B1) / RowGeom<B2>::R;
    const double nh = (double)nlimbs * (1u << (B1 + B2 - 1)), nb = (double)nlimbs * (8u << (B1 + B2));
    const double f = f64_share(L, t.ls);
    KLAUNCH(L, "ntt_inv_rows", nttw(nh * B2, f, 0, 2 * nb), (k_inv_rows<B2><<<nlimbs * g2, 128, 0, L.st>>>(t, perm, *L.tb, g2)));
    const u32 g1 = (1u << B2) / COLS;
    if (f == 1.0 && B1 >= 6)  // every limb FP64-mode: radix-16 columns
        inv_cols_r16_launch<B1, B2>(L, t, nlimbs, nttw(nh * B1, f, 2 * nh, 2 * nb));
    else
        KLAUNCH(L, "ntt_inv_cols", nttw(nh * B1, f, 2 * nh, 2 * nb), (k_inv_cols<B1, B2><<<nlimbs * g1, COLS * (1 << B1) / 8, 0, L.st>>>(t, *L.tb, g1)));
}

// Column launches over targets of both arithmetic classes: one mixed launch keeps integer- and
// FP64-mode CTAs side by side on every SM (their pipes run concurrently), single-class launches
// use fewer registers (more resident CTAs).  Measured: mixed wins at C4 (2 of 5 targets
// integer, 338 vs 343 ms/step), split wins at C3 (1 of 31, HMult 758 -> 743 us) -> split when
// at most 1/8 of the targets are integer-mode.  CKKS_SPLIT_CLASSES=0/1 forces either.
bool split_classes(const Launch &L, u32 n_int, u32 n_all)
{
    const char *e = std::getenv("CKKS_SPLIT_CLASSES");
    if (e) return std::atoi(e) != 0;
    return n_int * 8 <= n_all;
}

template <int B1, int B2>
void bcast_impl(const Launch &L, const TaskBcastCol &t, const SubMulArgs &a0, u32 nlimbs)
{
    SubMulArgs a = a0;
    int &s_raw = a.s_raw;
    const u32 g1 = (1u << B2) / COLS;
    const double nh = (double)nlimbs * (1u << (B1 + B2 - 1)), nb = (double)nlimbs * (8u << (B1 + B2));
    const double f = f64_share_range(L, t.toff, t.nt);
    u32 n_int = 0;
    for (u32 x = t.toff; x < t.toff + t.nt; ++x) n_int += f64_prime(L, x) ? 0 : 1;
    if (!split_classes(L, n_int, t.nt)) {
        KLAUNCH(L, "bcast_cols", nttw(nh * B1, f, 0, 2 * nb), (k_fwd_cols<B1, B2, TaskBcastCol><<<nlimbs * g1, COLS * (1 << B1) / 8, 0, L.st>>>(t, *L.tb, g1)));
    } else {  // one launch per run of targets of one arithmetic class
        const u32 np = nlimbs / t.nt;
        u32 a0 = t.toff;
        while (a0 < t.toff + t.nt) {
            const bool fc = f64_prime(L, a0);
            u32 e = a0 + 1;
            while (e < t.toff + t.nt && f64_prime(L, e) == fc) ++e;
            TaskBcastCol tr = t;
            tr.toff = a0;
            tr.nt = e - a0;
            tr.fnt = make_fdiv(e - a0);
            tr.ltoff = t.toff;
            tr.lnt = t.nt;
            const double nl = (double)np * (e - a0);
            const Work w = nttw(nl * (1u << (B1 + B2 - 1)) * B1, fc ? 1.0 : 0.0, 0, 2 * nl * (8u << (B1 + B2)));
            const u32 nli = np * (e - a0);
            if (fc && B1 >= 6 && (!tr.T || tr.qlcf)) {  // radix-16, lazy-double S rows
                KLAUNCH(L, "bcast_cols", w, (k_fwd_cols_r16<(B1 >= 6 ? B1 : 6), B2, TaskBcastCol><<<nli * g1, 1 << B1, 0, L.st>>>(tr, *L.tb, g1)));
                s_raw = 1;
            } else if (fc)
                KLAUNCH(L, "bcast_cols", w, (k_fwd_cols_f64<B1, B2, TaskBcastCol><<<nli * g1, COLS * (1 << B1) / 8, 0, L.st>>>(tr, *L.tb, g1)));
            else
                KLAUNCH(L, "bcast_cols", w, (k_fwd_cols<B1, B2, TaskBcastCol, 2><<<nli * g1, COLS * (1 << B1) / 8, 0, L.st>>>(tr, *L.tb, g1)));
            a0 = e;
        }
    }
    const u32 g2 = (1u << B1) / RowGeom<B2>::R;
    KLAUNCH(L, "submul_rows", nttw(nh * B2, f, 2 * nh, (a.base.base ? 4 : 3) * nb), (k_fwd_rows_submul<B2><<<nlimbs * g2, 128, 0, L.st>>>(a, *L.tb, g2)));
}

template <int B1, int B2>
void modup_impl(const Launch &L, const TaskModUpCol &t, u32 nlimbs)
{
    const u32 g1 = (1u << B2) / COLS;
    u32 diag = 0;  // (ciphertext, digit == target) slabs skipped
    for (u32 tl = 0; tl < t.T; ++tl) diag += (t.t0 + tl >= t.jw0 && t.t0 + tl < t.jw0 + t.nj) ? 1 : 0;
    const double live = (double)nlimbs - (double)(nlimbs / (t.T * t.nj)) * diag;
    const double nh = live * (1u << (B1 + B2 - 1)), nb = live * (8u << (B1 + B2));
    double fw = 0, wt = 0;  // targets weighted by their live digits
    for (u32 tl = 0; tl < t.T; ++tl) {
        const u32 tt = t.t0 + tl;
        const double live_t = (double)t.nj - (tt >= t.jw0 && tt < t.jw0 + t.nj ? 1 : 0);
        fw += f64_prime(L, tt < t.l ? tt : t.sp) ? live_t : 0;
        wt += live_t;
    }
    u32 n_int = 0;
    for (u32 x = t.t0; x < t.t0 + t.T; ++x) n_int += f64_prime(L, x < t.l ? x : t.sp) ? 0 : 1;
    if (!split_classes(L, n_int, t.T)) {
        KLAUNCH(L, "modup_cols", nttw(nh * B1, wt > 0 ? fw / wt : 0, 0, 2 * nb), (k_fwd_cols<B1, B2, TaskModUpCol><<<nlimbs * g1, COLS * (1 << B1) / 8, 0, L.st>>>(t, *L.tb, g1)));
        return;
    }
    // one launch per run of targets of one arithmetic class (single-path kernels).  With both
    // classes present the integer run (the 60-bit targets) goes to the second stream, beside the
    // FP64 run: its slabs are read only by the integer inner-product run, which mac_impl also puts
    // on that stream, and mac_impl's join orders everything before the next chunk (no join here)
    const u32 cnt = nlimbs / (t.T * t.nj);
    const bool fork = n_int > 0 && n_int < t.T && L.aux && !(L.prof && L.prof->on);
    if (fork) {
        cudaEventRecord(L.ev_fork, L.st);
        cudaStreamWaitEvent(L.aux, L.ev_fork, 0);
    }
    u32 a = t.t0;
    while (a < t.t0 + t.T) {
        const bool f = f64_prime(L, a < t.l ? a : t.sp);
        u32 e = a + 1;
        while (e < t.t0 + t.T && f64_prime(L, e < t.l ? e : t.sp) == f) ++e;
        Launch Lr = L;
        if (fork && !f) Lr.st = L.aux;
        TaskModUpCol tr = t;
        tr.t0 = a;
        tr.T = e - a;
        tr.fT = make_fdiv(e - a);
        tr.lt0 = t.t0;
        tr.lT = t.T;
        u32 dg = 0;
        for (u32 x = a; x < e; ++x) dg += (x >= t.jw0 && x < t.jw0 + t.nj) ? 1 : 0;
        const double lv = (double)cnt * ((double)(e - a) * t.nj - dg);
        const Work w = nttw(lv * (1u << (B1 + B2 - 1)) * B1, f ? 1.0 : 0.0, 0, 2 * lv * (8u << (B1 + B2)));
        const u32 nl = cnt * (e - a) * t.nj;
        if (f && B1 >= 6 && !std::getenv("CKKS_MODUP_R8"))  // radix-16 tile (CKKS_MODUP_R8=1: radix-8, A/B)
            KLAUNCH(Lr, "modup_cols", w, (k_fwd_cols_r16<(B1 >= 6 ? B1 : 6), B2, TaskModUpCol><<<nl * g1, 1 << B1, 0, Lr.st>>>(tr, *L.tb, g1)));
        else if (f)
            KLAUNCH(Lr, "modup_cols", w, (k_fwd_cols_f64<B1, B2, TaskModUpCol><<<nl * g1, COLS * (1 << B1) / 8, 0, Lr.st>>>(tr, *L.tb, g1)));
        else
            KLAUNCH(Lr, "modup_cols", w, (k_fwd_cols<B1, B2, TaskModUpCol, 2><<<nl * g1, COLS * (1 << B1) / 8, 0, Lr.st>>>(tr, *L.tb, g1)));
        a = e;
    }
}

// ext[c][p][t] = sum_s part[s][c][p][t - t0] mod q_t  (digit-split key switch, see MacArgs)
__global__ void __launch_bounds__(256) k_ks_split_sum(const u64 *part, u32 S, u32 cnt, u32 T, u32 t0, u32 l, u32 sp,
                                                      u64 *ext, u32 log_n, const ModC *mods)
{
    const size_t per = (size_t)cnt * 2 * T << log_n, nn = (size_t)1 << log_n;
    for (size_t x = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; x < per; x += (size_t)gridDim.x * blockDim.x * 2) {
        const size_t slab = x >> log_n, idx = x & (nn - 1);
        const u32 tl = (u32)(slab % T), cp = (u32)(slab / T);  // cp = c * 2 + p
        const u32 t = t0 + tl;
        const u64 q = mods[t < l ? t : sp].q;
        u64 s0 = 0, s1 = 0;
        for (u32 y = 0; y < S; ++y) {
            const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(part + y * per + x);
            s0 = addmod(s0, v.x, q);
            s1 = addmod(s1, v.y, q);
        }
        *reinterpret_cast<ulonglong2 *>(ext + (((size_t)cp * (l + 1) + t) << log_n) + idx) = make_ulonglong2(s0, s1);
    }
}

template <int B2>
bool mac_launch(const Launch &L, const MacArgs &a, u32 nct, int cls);

// ks_mac classes whose row-phase NTT runs on the FP64 pipe (3, 4, 5); 0-2, 6, 7 are integer
constexpr bool cls_f64(int c) { return c == 5; }

int ksmac_int_mode()  // CKKS_KSMAC_INT=1: integer classes on the original double-buffered body
{
    const char *e = std::getenv("CKKS_KSMAC_INT");
    return e ? std::atoi(e) : 0;
}

// split the target range into runs of one arithmetic class (see k_ks_mac)
template <int B2>
bool mac_impl(const Launch &L, const MacArgs &a0, u32 nct)
{
    const u32 cnt = nct / a0.T;
    auto cls_of = [&](u32 t) {
        const u64 q = L.hprimes[(t < a0.l) ? t : a0.sp];
        if (q < L.tb->f64_qmax) {
            // FP64 inner product (5): each term is reduced (|term| < 1.5 q), so the double
            // accumulator stays exact (< 1.5 l q < 2^50 for every supported l); the ModUp slabs
            // of FP64-mode targets hold lazy doubles that only this class reads
            return 5;
        }
        // CLS 1 (lazy row phase): q < 2^48, or a wide prime whose B2-stage phase fits (lazy_wide;
        // its phase-1 slab is canonical then)
        const int c = (a0.l >= 12 && q < (1ull << 40)) ? 2 : ((q < LAZY_Q_MAX || lazy_wide<B2>(q)) ? 1 : 0);
        if (c != 2 && ksmac_int_mode() != 1) return c == 1 ? 6 : 7;  // the CLS 5-style pipeline
        return c;
    };
    struct Run {
        MacArgs a;
        int cls;
    };
    Run runs[64];
    int nr = 0;
    bool any_f64 = false, any_int = false;
    u32 t = a0.t0;
    while (t < a0.t0 + a0.T && nr < 64) {
        const int c = cls_of(t);
        u32 e = t + 1;
        while (e < a0.t0 + a0.T && cls_of(e) == c) ++e;
        runs[nr] = Run{a0, c};
        runs[nr].a.t0 = t;
        runs[nr].a.T = e - t;
        ++nr;
        (cls_f64(c) ? any_f64 : any_int) = true;
        t = e;
    }
    // FP64-pipe and integer-pipe classes run concurrently on two streams so their CTAs share
    // the SMs (each class leaves the other's pipe idle)
    // (not while profiling: per-launch CUDA events on two concurrent streams would each count
    // the other's co-running time; the profiled pass measures the kernels serially, as ncu does)
    const bool fork = any_f64 && any_int && L.aux && !(L.prof && L.prof->on);
    if (fork) {
        cudaEventRecord(L.ev_fork, L.st);
        cudaStreamWaitEvent(L.aux, L.ev_fork, 0);
    }
    bool pinv_done = false;
    for (int r = 0; r < nr; ++r) {
        Launch Lr = L;
        MacArgs ar = runs[r].a;
        if (fork) {  // the two streams' digit-split launches use disjoint halves of the scratch
            Lr.split_words = L.split_words / 2;
            if (!cls_f64(runs[r].cls)) {
                Lr.st = L.aux;
                Lr.split = L.split ? L.split + Lr.split_words : nullptr;
            }
        }
        pinv_done |= mac_launch<B2>(Lr, ar, cnt * ar.T, runs[r].cls);
    }
    if (fork) {
        cudaEventRecord(L.ev_join, L.aux);
        cudaStreamWaitEvent(L.st, L.ev_join, 0);
    }
    return pinv_done;
}

template <int B2>
bool mac_launch(const Launch &L, const MacArgs &a0, u32 nct, int cls)
{
    MacArgs a = a0;
    a.fT = make_fdiv(a.T);
    const bool has_p = a.t0 + a.T > a.l;  // this run includes the special-prime target
    if (!(cls == 6 || cls == 7) || !has_p) a.pinv_rows = 0;
    const u32 log_n = L.tb->log_n;
    const u32 g = (1u << (log_n - B2)) / MacGeom<B2>::R;
    const u32 cnt = nct / a.T;
    const u32 nd = a.halpha ? a.nd : a.l;
    const u32 jb = a.jw0, je = a.jw1 ? a.jw1 : nd, nj = je - jb;
    u32 diag = 0;
    for (u32 tl = 0; tl < a.T; ++tl) {
        const u32 t = a.t0 + tl, td = a.halpha ? (t < a.l ? t / a.halpha : ~0u) : t;
        diag += (td >= jb && td < je) ? 1 : 0;
    }
    const double n_ = (double)(1u << log_n);
    const double ntts = (double)cnt * ((double)a.T * nj - diag);
    // bytes: phase-1 slabs in, d limbs for diagonal digits, key (once per launch), 2 outputs
    const double bytes = 8.0 * n_ * (ntts + (double)cnt * diag + 2.0 * a.T * nj + 2.0 * cnt * a.T * (a.accum ? 2 : 1));
    Work w = nttw(ntts * n_ / 2 * B2, cls_f64(cls) ? 1.0 : 0.0, 2.0 * cnt * a.T * nj * n_, bytes);
    if (cls == 5) a.kcomp = L.key_compact ? 1 : 0;
    if (a.kcomp) w.bytes -= 8.0 * n_ * (2.0 * a.T * nj) * 3.0 / 8.0;  // key rows read as 5 of 8 bytes
    if (cls == 5) {  // inner product on the FP64 pipe
        w.fmac = w.mac;
        w.mac = 0;
    }
    // a launch too small to fill the GPU (e.g. the special-prime target of one ciphertext at
    // N = 2^16: 128 CTAs of 2 warps, each looping over all l digits) splits its digit loop over
    // gridDim.y CTA rows and sums the partial results in k_ks_split_sum
    u32 S = 1;
    const u32 ctas = nct * g, want = 8 * L.n_sm;
    if (L.split && !a.halpha && a.l >= 8 && ctas * 2 <= want && !a.jw1 && !a.accum) {
        S = std::min<u32>((want + ctas - 1) / ctas, a.l / 4);
        if (S >= 2) {
            a.jper = (a.l + S - 1) / S;
            S = (a.l + a.jper - 1) / a.jper;
        }
        if (S < 2 || (size_t)S * cnt * 2 * a.T << log_n > L.split_words) S = 1;
        if (S > 1) {
            a.part = L.split;
            a.cnt_run = cnt;
        }
    }
    if (a.pinv_rows && S == 1) {  // + the special-prime limb's INTT row phase (both polynomials)
        const double ib = (double)cnt * 2 * (n_ / 2) * B2;
        (L.hprimes[a.sp] < L.tb->f64_qmax ? w.fbfly : w.bfly) += ib;
    }
    const dim3 grid(nct * g, S);
    if (cls == 5)
        KLAUNCH(L, "ks_mac", w, (k_ks_mac<B2, 5><<<grid, 64, 0, L.st>>>(a, *L.tb, g)));
    else if (cls == 6)
        KLAUNCH(L, "ks_mac", w, (k_ks_mac<B2, 6><<<grid, 64, 0, L.st>>>(a, *L.tb, g)));
    else if (cls == 7)
        KLAUNCH(L, "ks_mac", w, (k_ks_mac<B2, 7><<<grid, 64, 0, L.st>>>(a, *L.tb, g)));
    else if (cls == 2)
        KLAUNCH(L, "ks_mac", w, (k_ks_mac<B2, 2><<<grid, 64, 0, L.st>>>(a, *L.tb, g)));
    else if (cls == 1)
        KLAUNCH(L, "ks_mac", w, (k_ks_mac<B2, 1><<<grid, 64, 0, L.st>>>(a, *L.tb, g)));
    else
        KLAUNCH(L, "ks_mac", w, (k_ks_mac<B2, 0><<<grid, 64, 0, L.st>>>(a, *L.tb, g)));
    if (S > 1) {
        const size_t per = (size_t)cnt * 2 * a.T << log_n;
        const u32 blocks = (u32)std::min<size_t>((per / 2 + 255) / 256, (size_t)L.n_sm * 8);
        KLAUNCH(L, "ks_split_sum", (Work{0, 0, 8.0 * per * (S + 1), 0}),
                (k_ks_split_sum<<<blocks, 256, 0, L.st>>>(L.split, S, cnt, a.T, a.t0, a.l, a.sp, a.ext, log_n,
                                                         L.tb->mod)));
    }
    return a.pinv_rows && S == 1;
}

#define CKKS_DISPATCH_LOGN(LOGN, CALL)             \
    switch (LOGN) {                                \
    case 10: CALL(5, 5); break;                    \
    case 11: CALL(5, 6); break;                    \
    case 12: CALL(6, 6); break;                    \
    case 13: CALL(6, 7); break;                    \
    case 14: CALL(7, 7); break;                    \
    case 15: CALL(7, 8); break;                    \
    case 16: CALL(8, 8); break;                    \
    default: break;                                \
    }

}  // namespace

void launch_ntt_fwd(const Launch &L, PolyMap src, PolyMap dst, u32 npolys, LimbSet ls)
{
    if (!npolys || !ls.n) return;
    TaskPlainCol t{src, dst, ls, L.tb->log_n, make_fdiv(ls.n)};
    const u32 nl = npolys * ls.n;
#define CALLF(b1, b2) ntt_fwd_impl<b1, b2>(L, t, nl)
    CKKS_DISPATCH_LOGN(L.tb->log_n, CALLF)
#undef CALLF
}

namespace {
template <int B1, int B2>
void tensor_rows_impl(const Launch &L, const TensorRows &t, u32 cnt)
{
    const u32 g2 = (1u << B1) / RowGeom<B2>::R;
    const u32 nl = cnt * t.l;
    const double nh = (double)nl * (1u << (B1 + B2 - 1)), nb = (double)nl * (8u << (B1 + B2));
    const double f = f64_share(L, LimbSet{t.l, t.l, 0, 0});
    Work w = nttw(nh * B2, f, 2 * nh * 4, 9 * nb);  // 4 products per coefficient; 4 in, 5 out
    if (f > 0) {  // the tensor's products on the FP64 pipe (FP64-mode limbs)
        w.fmac += w.mac * f;
        w.mac *= 1 - f;
    }
    KLAUNCH(L, "tensor_inv_rows", w, (k_tensor_inv_rows<B2><<<nl * g2, 128, 0, L.st>>>(t, *L.tb, g2)));
}
template <int B1, int B2>
void ntt_inv_cols_impl(const Launch &L, const TaskPlainCol &t, u32 nlimbs)
{
    const u32 g1 = (1u << B2) / COLS;
    const double nh = (double)nlimbs * (1u << (B1 + B2 - 1)), nb = (double)nlimbs * (8u << (B1 + B2));
    const double f = f64_share(L, t.ls);
    if (f == 1.0 && B1 >= 6)  // every limb FP64-mode: radix-16 columns
        inv_cols_r16_launch<B1, B2>(L, t, nlimbs, nttw(nh * B1, f, 2 * nh, 2 * nb));
    else
        KLAUNCH(L, "ntt_inv_cols", nttw(nh * B1, f, 2 * nh, 2 * nb), (k_inv_cols<B1, B2><<<nlimbs * g1, COLS * (1 << B1) / 8, 0, L.st>>>(t, *L.tb, g1)));
}
}  // namespace

void launch_tensor_inv_rows(const Launch &L, PolyMap a, PolyMap b, PolyMap out, PolyMap d2, PolyMap dr, u32 nct, u32 l)
{
    if (!nct || !l) return;
    TensorRows t{a, b, out, d2, dr, l, make_fdiv(l)};
#define CALLTR(b1, b2) tensor_rows_impl<b1, b2>(L, t, nct)
    CKKS_DISPATCH_LOGN(L.tb->log_n, CALLTR)
#undef CALLTR
}

void launch_ntt_inv_cols(const Launch &L, PolyMap data, u32 npolys, LimbSet ls)
{
    if (!npolys || !ls.n) return;
    TaskPlainCol t{data, data, ls, L.tb->log_n, make_fdiv(ls.n)};
#define CALLIC(b1, b2) ntt_inv_cols_impl<b1, b2>(L, t, npolys * ls.n)
    CKKS_DISPATCH_LOGN(L.tb->log_n, CALLIC)
#undef CALLIC
}

void launch_ntt_inv(const Launch &L, PolyMap src, PolyMap dst, u32 npolys, LimbSet ls, const u32 *perm)
{
    if (!npolys || !ls.n) return;
    TaskPlainCol t{src, dst, ls, L.tb->log_n, make_fdiv(ls.n)};
    const u32 nl = npolys * ls.n;
#define CALLI(b1, b2) ntt_inv_impl<b1, b2>(L, t, nl, perm)
    CKKS_DISPATCH_LOGN(L.tb->log_n, CALLI)
#undef CALLI
}

namespace {
template <int B1, int B2>
void inv_modup_impl(const Launch &L, const TaskPlainCol &t, u32 nlimbs, const u32 *perm, u64 *I, u32 l, u32 t0,
                    u32 T, u32 sp, bool rows_done)
{
    const u32 g2 = (1u << B1) / RowGeom<B2>::R;
    const double nh = (double)nlimbs * (1u << (B1 + B2 - 1)), nb = (double)nlimbs * (8u << (B1 + B2));
    const double f = f64_share(L, t.ls);
    if (!rows_done)  // (else t.dst already holds the row-phase output: launch_tensor_inv_rows)
        KLAUNCH(L, "ntt_inv_rows", nttw(nh * B2, f, 0, 2 * nb), (k_inv_rows<B2><<<nlimbs * g2, 128, 0, L.st>>>(t, perm, *L.tb, g2)));
    const u32 g1 = (1u << B2) / COLS;
    const u32 cnt = nlimbs / l;
    double fw = 0, wt = 0;  // ModUp column phases by class (as modup_impl)
    u32 diag = 0;
    for (u32 tl = 0; tl < T; ++tl) {
        const u32 tt = t0 + tl;
        const double live_t = (double)l - (tt < l ? 1 : 0);
        diag += (tt < l) ? 1 : 0;
        fw += f64_prime(L, tt < l ? tt : sp) ? live_t : 0;
        wt += live_t;
    }
    const double live = (double)cnt * ((double)T * l - diag);
    const double nhm = live * (1u << (B1 + B2 - 1)), nbm = live * (8u << (B1 + B2));
    Work w = nttw(nh * B1, f, 2 * nh, 2 * nb);  // the digits' inverse column phase
    const Work wm = nttw(nhm * B1, wt > 0 ? fw / wt : 0, 0, nbm);
    w.bfly += wm.bfly;
    w.fbfly += wm.fbfly;
    w.bytes = nb + nbm;  // row-phase output in once, ModUp slabs out
    const InvModUpArgs a{t, I, l, t0, T, sp};
    KLAUNCH(L, "inv_modup_cols", w, (k_inv_cols_modup<B1, B2><<<nlimbs * g1, COLS * (1 << B1) / 8, 0, L.st>>>(a, *L.tb, g1)));
}
}  // namespace

void launch_inv_modup(const Launch &L, PolyMap src, u64 *Dtmp, u32 cnt, u32 l, const u32 *perm, u32 t0, u32 T,
                      u64 *I, u32 sp, bool rows_done)
{
    if (!cnt || !l) return;
    const LimbSet ls{l, l, 0, sp};
    TaskPlainCol t{src, PolyMap{Dtmp, l}, ls, L.tb->log_n, make_fdiv(l)};
    const u32 nl = cnt * l;
#define CALLIM(b1, b2) inv_modup_impl<b1, b2>(L, t, nl, perm, I, l, t0, T, sp, rows_done)
    CKKS_DISPATCH_LOGN(L.tb->log_n, CALLIM)
#undef CALLIM
}

namespace {
template <int B1, int B2>
void inv_bcast_impl(const Launch &L, const TaskPlainCol &t, const SubMulArgs &sa, u32 npolys, bool rows_done)
{
    const u32 g2 = (1u << B1) / RowGeom<B2>::R, g1 = (1u << B2) / COLS;
    const double n1 = (double)npolys * (1u << (B1 + B2 - 1)), nb1 = (double)npolys * (8u << (B1 + B2));
    const double fs = f64_share(L, t.ls);
    if (!rows_done)  // (else the key-switch inner product already applied the inverse row phase)
        KLAUNCH(L, "ntt_inv_rows", nttw(n1 * B2, fs, 0, 2 * nb1), (k_inv_rows<B2><<<npolys * g2, 128, 0, L.st>>>(t, nullptr, *L.tb, g2)));
    const double ft = f64_share_range(L, sa.toff, sa.nt);
    const double nl = (double)npolys * sa.nt;
    Work w = nttw(n1 * B1, fs, n1 * 2, nb1);  // the source limb's inverse column phase
    const Work wb = nttw(nl * (1u << (B1 + B2 - 1)) * B1, ft, 0, nl * (8u << (B1 + B2)));
    w.bfly += wb.bfly;
    w.fbfly += wb.fbfly;
    w.bytes += wb.bytes;
    const InvBcastArgs a{t, const_cast<u64 *>(sa.S), sa.nt, sa.toff};
    KLAUNCH(L, "inv_bcast_cols", w, (k_inv_cols_bcast<B1, B2><<<npolys * g1, COLS * (1 << B1) / 8, 0, L.st>>>(a, *L.tb, g1)));
    const u32 nlimbs = npolys * sa.nt;
    const double nh = (double)nlimbs * (1u << (B1 + B2 - 1)), nb = (double)nlimbs * (8u << (B1 + B2));
    KLAUNCH(L, "submul_rows", nttw(nh * B2, ft, 2 * nh, (sa.base.base ? 4 : 3) * nb), (k_fwd_rows_submul<B2><<<nlimbs * g2, 128, 0, L.st>>>(sa, *L.tb, g2)));
}
}  // namespace

void launch_inv_bcast_submul(const Launch &L, PolyMap src, PolyMap tmp, LimbSet ls, u32 npolys, u32 nt, u32 toff,
                             u64 *scratch, PolyMap x, PolyMap out, const ulonglong2 *consts, PolyMap base,
                             const u32 *base_perm, bool base_c0_only, PolyMap acc, bool rows_done)
{
    if (!npolys || !nt) return;
    TaskPlainCol t{src, tmp, ls, L.tb->log_n, make_fdiv(ls.n)};
    SubMulArgs a{scratch, nt, toff, x, out, base, acc, base_perm, base_c0_only ? 1 : 0, consts};
#define CALLIB(b1, b2) inv_bcast_impl<b1, b2>(L, t, a, npolys, rows_done)
    CKKS_DISPATCH_LOGN(L.tb->log_n, CALLIB)
#undef CALLIB
}

void launch_bcast_submul(const Launch &L, const u64 *X, u32 x_stride, u32 x_prime, u32 npolys, u32 nt, u32 toff,
                         u64 *scratch, PolyMap x, PolyMap out, const ulonglong2 *consts, PolyMap base,
                         const u32 *base_perm, bool base_c0_only, PolyMap acc, const u64 *T,
                         const ulonglong2 *qlc, const ulonglong2 *bconsts, const double2 *qlcf)
{
    if (!npolys || !nt) return;
    TaskBcastCol t{X, scratch, nt, x_prime, x_stride, L.tb->log_n, toff, make_fdiv(nt)};
    t.T = T;
    t.qlc = qlc;
    t.qlcf = qlcf;
    SubMulArgs a{scratch, nt, toff, x, out, base, acc, base_perm, base_c0_only ? 1 : 0, consts};
    a.bconsts = bconsts;
#define CALLB(b1, b2) bcast_impl<b1, b2>(L, t, a, npolys * nt)
    CKKS_DISPATCH_LOGN(L.tb->log_n, CALLB)
#undef CALLB
}

void launch_ks_modup_cols(const Launch &L, const u64 *D, u32 dw, u32 dcnt, u32 c0, u32 l, u32 cnt, u32 t0, u32 T,
                          u64 *I, u32 sp, u32 jw0, u32 nj)
{
    const u32 jn = nj ? nj : l;
    TaskModUpCol t{D, I, l, t0, T, sp, L.tb->log_n, dw, dcnt, c0, make_fdiv(T), make_fdiv(jn)};
    t.jw0 = nj ? jw0 : 0;
    t.nj = jn;
#define CALLM(b1, b2) modup_impl<b1, b2>(L, t, cnt * T * jn)
    CKKS_DISPATCH_LOGN(L.tb->log_n, CALLM)
#undef CALLM
}

bool launch_ks_mac(const Launch &L, const u64 *I, PolyMap din, const u32 *perm, const u64 *key, u32 Lk, u32 l,
                   u32 cnt, u32 t0, u32 T, u64 *ext, u32 sp, bool p_inv_rows, u32 jw0, u32 jw1, bool accum,
                   u32 lay_t0, u32 lay_T)
{
    MacArgs a{I, din, perm, key, ext, Lk, l, t0, T, sp, lay_T ? lay_t0 : t0, lay_T ? lay_T : T};
    a.pinv_rows = p_inv_rows ? 1 : 0;
    a.jw0 = jw0;
    a.jw1 = jw1;
    a.accum = accum ? 1 : 0;
    bool done = false;
#define CALLK(b1, b2) done = mac_impl<b2>(L, a, cnt * T)
    CKKS_DISPATCH_LOGN(L.tb->log_n, CALLK)
#undef CALLK
    return done;
}

void launch_addsub(const Launch &L, PolyMap a, PolyMap b, PolyMap out, u32 npolys, u32 l, int op)
{
    run_elem(L, FAddSub{a, b, out, op}, npolys, l);
}
void launch_mul_poly(const Launch &L, PolyMap a, PolyMap b, u32 b_div, u32 b_mod, PolyMap out, u32 npolys, u32 l)
{
    run_elem(L, FMulPoly{a, b, out, b_div, b_mod}, npolys, l);
}
void launch_add_plain(const Launch &L, PolyMap ct, PolyMap pt, u32 pt_bcast, PolyMap out, u32 nct, u32 l)
{
    run_elem(L, FAddPlain{ct, pt, out, pt_bcast}, 2 * nct, l);
}
void launch_mul_scalar(const Launch &L, PolyMap a, PolyMap out, u32 npolys, u32 l, const ulonglong2 *consts)
{
    run_elem(L, FMulScalar{a, out, consts}, npolys, l);
}
void launch_add_scalar_c0(const Launch &L, PolyMap ct, PolyMap out, u32 nct, u32 l, const u64 *consts)
{
    run_elem(L, FAddScalarC0{ct, out, consts}, 2 * nct, l);
}
void launch_tensor(const Launch &L, PolyMap a, PolyMap b, PolyMap out, PolyMap d2, u32 nct, u32 l, u32 adiv, u32 amod,
                   u32 bdiv, u32 bmod)
{
    run_elem(L, FTensor{a, b, out, d2, adiv, amod, bdiv, bmod, L.tb->psif, L.tb->f64_qmax}, nct, l);
}
void launch_from_signed(const Launch &L, const int64_t *e, PolyMap out, u32 npolys, LimbSet ls)
{
    // limbs are table-indexed 0..ls.n-1 (contiguous q's then P), see LimbSet usage in ckks.cu
    run_elem(L, FFromSigned{e, out}, npolys, ls.n);
}
void launch_copy(const Launch &L, PolyMap src, PolyMap dst, u32 npolys, u32 l)
{
    run_elem(L, FCopy{src, dst}, npolys, l);
}
void launch_permute(const Launch &L, PolyMap src, PolyMap dst, u32 npolys, u32 l, const u32 *perm)
{
    run_elem(L, FPermute{src, dst, perm}, npolys, l);
}
void launch_keygen_b(const Launch &L, const u64 *a, const u64 *e, const u64 *s, const u64 *sfrom, const u64 *pmod,
                     u64 *key, u32 Lk, u32 K, u32 alpha, u32 dnum)
{
    run_elem(L, FKeygenB{a, e, s, sfrom, pmod, key, Lk, K, alpha}, dnum, Lk + K);
}
void launch_mul_add(const Launch &L, PolyMap a, PolyMap s, u32 s_bcast, PolyMap b, PolyMap out, u32 npolys, u32 l,
                    int negate_prod)
{
    run_elem(L, FMulAdd{a, s, b, out, s_bcast, negate_prod}, npolys, l);
}
void launch_modadd_gathered(const Launch &L, const u64 *g, size_t stride_words, u32 R, PolyMap out, u32 npolys,
                            u32 l)
{
    run_elem(L, FModAddGathered{g, stride_words, R, out}, npolys, l);
}

// ------------------------------------------------------------------------------------
// PrivFT chunk-dot: per coefficient position a small modular matrix product
// out[b][jj] = sum_k C[b][k] * H[jj][k].  One thread = one position and a BT x JT
// output tile (x 2 polynomials) held as 128-bit accumulators; consecutive CTAs walk the
// tiles of one position block so C and H for that block are re-read from L2, not HBM.
// ------------------------------------------------------------------------------------
namespace {
constexpr int CD_BT = 4, CD_JT = 4, CD_THREADS = 128;

template <class Acc>
__device__ __forceinline__ void chunkdot_body(const u64 *ct, u32 ct_cap, const u64 *pt, u32 pt_cap, u64 *out,
                                              u32 out_cap, u32 B, u32 J, u32 K, u32 i, u32 idx, size_t n,
                                              const ModC &m, u32 b0, u32 j0, u32 fold)
{
    // one pointer per stream, advanced by a constant stride per chunk k (no per-k index math)
    const u64 *hp[CD_JT], *cp[CD_BT];
#pragma unroll
    for (int y = 0; y < CD_JT; ++y) {
        const u32 jj = j0 + y < J ? j0 + y : J - 1;
        hp[y] = pt + (((size_t)jj * K) * pt_cap + i) * n + idx;
    }
#pragma unroll
    for (int x = 0; x < CD_BT; ++x) {
        const u32 b = b0 + x < B ? b0 + x : B - 1;
        cp[x] = ct + (((size_t)b * K) * 2 * ct_cap + i) * n + idx;
    }
    const size_t hs = (size_t)pt_cap * n, cs = (size_t)2 * ct_cap * n, c1 = (size_t)ct_cap * n;
    Acc acc[CD_BT][CD_JT][2];
    // `fold` terms (each < q^2) plus one folded residue (< q) stay below the accumulator's
    // capacity; longer sums are reduced mod q every `fold` chunks (exact: the accumulator is
    // replaced by its residue).
    for (u32 kb = 0; kb < K; kb += fold) {
    if (kb) {
#pragma unroll
        for (int x = 0; x < CD_BT; ++x)
#pragma unroll
            for (int y = 0; y < CD_JT; ++y) {
                acc[x][y][0].fold(m);
                acc[x][y][1].fold(m);
            }
    }
    const u32 kend = K - kb < fold ? K : kb + fold;
    for (u32 k = kb; k < kend; ++k) {
        u64 h[CD_JT], c0[CD_BT], cc1[CD_BT];
#pragma unroll
        for (int y = 0; y < CD_JT; ++y) {
            h[y] = __ldg(hp[y]);
            hp[y] += hs;
        }
#pragma unroll
        for (int x = 0; x < CD_BT; ++x) {
            c0[x] = __ldg(cp[x]);
            cc1[x] = __ldg(cp[x] + c1);
            cp[x] += cs;
        }
#pragma unroll
        for (int x = 0; x < CD_BT; ++x)
#pragma unroll
            for (int y = 0; y < CD_JT; ++y) {
                acc[x][y][0].mac(c0[x], h[y]);
                acc[x][y][1].mac(cc1[x], h[y]);
            }
    }
    }
#pragma unroll
    for (int x = 0; x < CD_BT; ++x)
#pragma unroll
        for (int y = 0; y < CD_JT; ++y) {
            const u32 b = b0 + x, jj = j0 + y;
            if (b < B && jj < J) {
                const size_t o = (((size_t)b * J + jj) * 2 * out_cap + i) * n + idx;
                out[o] = acc[x][y][0].reduce(m);
                out[o + (size_t)out_cap * n] = acc[x][y][1].reduce(m);
            }
        }
}

__global__ void __launch_bounds__(CD_THREADS) k_chunkdot(const u64 *ct, u32 ct_cap, const u64 *pt, u32 pt_cap,
                                                       u64 *out, u32 out_cap, u32 B, u32 J, u32 K, u32 l,
                                                       u32 log_n, const ModC *mods, u32 ntb)
{
    const u32 tile = blockIdx.x;
    const u32 bt = tile % ntb, jt = tile / ntb;
    const size_t pos = (size_t)blockIdx.y * CD_THREADS + threadIdx.x;  // (limb i, idx)
    const u32 i = (u32)(pos >> log_n), idx = (u32)(pos & ((1u << log_n) - 1));
    if (i >= l) return;
    const ModC m = load_mod(mods, i);
    const size_t n = (size_t)1 << log_n;
    // limb-uniform branch (a CTA lies inside one limb)
    if (m.q < (1ull << 40))
        chunkdot_body<Acc40>(ct, ct_cap, pt, pt_cap, out, out_cap, B, J, K, i, idx, n, m, bt * CD_BT, jt * CD_JT,
                             Acc40::MAX_TERMS);
    else
        chunkdot_body<Acc128>(ct, ct_cap, pt, pt_cap, out, out_cap, B, J, K, i, idx, n, m, bt * CD_BT, jt * CD_JT,
                              acc128_fold_terms(m.q));
}

struct FMulScalarPerCt {
    static constexpr const char *NAME = "elem_mulscalar_ct";
    static constexpr double MULS = 1, WORDS = 2;
    PolyMap a, out;
    const ulonglong2 *c;
    u32 l;
    __device__ void operator()(u32 p, u32 i, u32 idx, const ModC &m, u32 log_n) const
    {
        const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(limb_ptr(a, p, i, log_n) + idx);
        const ulonglong2 w = __ldg(c + (size_t)(p >> 1) * l + i);
        *reinterpret_cast<ulonglong2 *>(limb_ptr_w(out, p, i, log_n) + idx) =
            make_ulonglong2(shoup(x.x, w.x, w.y, m.q), shoup(x.y, w.x, w.y, m.q));
    }
};
}  // namespace

void launch_chunkdot(const Launch &L, const u64 *ct, u32 ct_cap, const u64 *pt, u32 pt_cap, u64 *out, u32 out_cap,
                     u32 B, u32 J, u32 K, u32 l)
{
    const u32 ntb = (B + CD_BT - 1) / CD_BT, ntj = (J + CD_JT - 1) / CD_JT;
    const size_t positions = (size_t)l << L.tb->log_n;
    dim3 grid(ntb * ntj, (unsigned)((positions + CD_THREADS - 1) / CD_THREADS));
    const double pos = (double)positions;
    KLAUNCH(L, "chunkdot", (Work{0, 2.0 * B * J * K * pos, 8.0 * pos * (2.0 * B * K + (double)J * K + 2.0 * B * J)}),
            (k_chunkdot<<<grid, CD_THREADS, 0, L.st>>>(ct, ct_cap, pt, pt_cap, out, out_cap, B, J, K, l,
                                                                     L.tb->log_n, L.tb->mod, ntb)));
}

void launch_mul_scalar_per_ct(const Launch &L, PolyMap a, PolyMap out, u32 nct, u32 l, const ulonglong2 *consts)
{
    run_elem(L, FMulScalarPerCt{a, out, consts, l}, 2 * nct, l);
}

// ------------------------------------------------------------------------------------
// Hybrid key switching: alpha-limb digits, K special primes, HPS fast
// base conversion.  Extended-basis slots at level l: s < l -> q_s; s = l + k -> p_k.
// ------------------------------------------------------------------------------------
namespace {
constexpr int HYB_MAX_ALPHA = 16;

// X[c][d][s] (coefficient form) = conv_{D_d}(D[c]) mod m_s for s not in D_d
// yinv: [beta][alpha] (Shoup pairs) (Q_D/q_i)^{-1} mod q_i;  conv: [beta][alpha][ne] (Q_D/q_i) mod m_s
struct ModUpConvArgs {
    const u64 *D;  // [cnt][l][N]
    u64 *X;        // [cnt][beta][ne][N]
    const ulonglong2 *yinv;
    const u64 *conv;
    u32 l, L, K, alpha, beta, ne;
};

// two coefficients per thread (16-byte accesses); one digit's alpha residues are reduced
// once ([x_i (Q_D/q_i)^{-1}]_{q_i}, Shoup) and reused for every target slot.
template <class Acc>
__device__ __forceinline__ void conv_slot(const u64 (*y)[2], u32 ns, const u64 *cv, u32 stride, const ModC &m,
                                          u64 &o0, u64 &o1)
{
    Acc a0, a1;
#pragma unroll
    for (int i = 0; i < HYB_MAX_ALPHA; ++i)
        if (i < (int)ns) {
            const u64 w = __ldg(cv + (size_t)i * stride);
            a0.mac(y[i][0], w);
            a1.mac(y[i][1], w);
        }
    o0 = a0.reduce(m);
    o1 = a1.reduce(m);
}

constexpr u32 CONV_SLOTS = 8;  // target slots per thread (the digit's residues are re-reduced per chunk)

__global__ void __launch_bounds__(128) k_modup_conv(ModUpConvArgs a, const ModC *mods, u32 log_n, u32 cnt)
{
    const size_t n = (size_t)1 << log_n;
    const u32 nsc = (a.ne + CONV_SLOTS - 1) / CONV_SLOTS;
    const size_t gid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t pairs = (size_t)cnt * a.beta * (n >> 1);
    if (gid >= pairs * nsc) return;
    const u32 sc = (u32)(gid / pairs);  // slot chunk (outermost: a warp shares it)
    const size_t e2 = (gid % pairs) << 1;
    const u32 idx = (u32)(e2 & (n - 1));
    const u32 d = (u32)((e2 >> log_n) % a.beta), c = (u32)((e2 >> log_n) / a.beta);
    const u32 lo = d * a.alpha, hi = min(lo + a.alpha, a.l), ns = hi - lo;
    u64 y[HYB_MAX_ALPHA][2];
    bool small = true;  // every digit prime < 2^40 (Acc40 precondition on the inputs)
#pragma unroll
    for (int i = 0; i < HYB_MAX_ALPHA; ++i) {
        if (i < (int)ns) {
            const ModC m = load_mod(mods, lo + i);
            small = small && m.q < (1ull << 40);
            const ulonglong2 w = __ldg(a.yinv + (size_t)d * a.alpha + i);
            const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(a.D + ((size_t)c * a.l + lo + i) * n + idx);
            y[i][0] = shoup(x.x, w.x, w.y, m.q);
            y[i][1] = shoup(x.y, w.x, w.y, m.q);
        }
    }
    const u64 *cv = a.conv + (size_t)d * a.alpha * a.ne;
    u64 *xo = a.X + (((size_t)c * a.beta + d) * a.ne) * n + idx;
    const u32 s_end = min(a.ne, (sc + 1) * CONV_SLOTS);
    for (u32 s = sc * CONV_SLOTS; s < s_end; ++s) {
        if (s >= lo && s < hi) continue;
        const u32 prime = s < a.l ? s : a.L + (s - a.l);
        const ModC m = load_mod(mods, prime);
        u64 o0, o1;
        if (small && m.q < (1ull << 40))
            conv_slot<Acc40>(y, ns, cv + s, a.ne, m, o0, o1);
        else
            conv_slot<Acc128>(y, ns, cv + s, a.ne, m, o0, o1);
        *reinterpret_cast<ulonglong2 *>(xo + (size_t)s * n) = make_ulonglong2(o0, o1);
    }
}

// ModUp fast base conversion, v2: one thread = 2 coefficients of one digit and a chunk of
// target slots.  The digit's alpha residues are reduced once ([x_i (Q_D/q_i)^{-1}]_{q_i},
// Shoup) and kept as exact doubles when every digit prime is FP64-mode; FP64-mode target
// slots then accumulate on the FP64 pipe (exact two-product terms |r| < 2.5 m_s summed in a
// double, < 2.5 alpha m_s < 2^50), integer-mode slots (the 60-bit special primes) in 128-bit
// integer accumulators.  Slot loop and class choice are warp-uniform.
template <int MAXA>
__global__ void __launch_bounds__(128) k_modup_conv2(ModUpConvArgs a, Tables tb, u32 nchunks, u32 chunk, int f64in)
{
    const ModC *mods = tb.mod;
    const u32 log_n = tb.log_n;
    const u32 n = 1u << log_n, per_cd = n >> 8;  // 256 coefficients per CTA
    u32 b = blockIdx.x;
    const u32 cb = b % per_cd;
    b /= per_cd;
    const u32 sc = b % nchunks;
    b /= nchunks;
    const u32 d = b % a.beta, c = b / a.beta;
    const u32 idx = (cb << 8) + 2 * threadIdx.x;
    const u32 lo = d * a.alpha, ns = min(a.alpha, a.l - lo);
    u64 y[MAXA][2];
#pragma unroll
    for (int i = 0; i < MAXA; ++i) {
        y[i][0] = y[i][1] = 0;
        if (i < (int)ns) {
            const ModC m = load_mod(mods, lo + i);
            const ulonglong2 w = __ldg(a.yinv + (size_t)d * a.alpha + i);
            const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(a.D + (((size_t)c * a.l + lo + i) << log_n) + idx);
            y[i][0] = shoup(x.x, w.x, w.y, m.q);
            y[i][1] = shoup(x.y, w.x, w.y, m.q);
        }
    }
    const u64 *cv = a.conv + (size_t)d * a.alpha * a.ne;
    u64 *xo = a.X + (((size_t)c * a.beta + d) * a.ne << log_n) + idx;
    const u32 s1 = min(a.ne, (sc + 1) * chunk);
    for (u32 s = sc * chunk; s < s1; ++s) {
        if (s >= lo && s < lo + ns) continue;  // the digit's own limbs are not converted
        const u32 prime = s < a.l ? s : a.L + (s - a.l);
        const ModC m = load_mod(mods, prime);
        ulonglong2 o;
        if (f64in && m.q < tb.f64_qmax) {
            const double2 qq = __ldg(tb.psif + ((size_t)prime << log_n));  // entry 0: (q, 1/q)
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int i = 0; i < MAXA; ++i)
                if (i < (int)ns) {
                    const double w = u2d(__ldg(cv + (size_t)i * a.ne + s));
                    a0 += f64_mac_term(u2d(y[i][0]), w, qq.x, qq.y);
                    a1 += f64_mac_term(u2d(y[i][1]), w, qq.x, qq.y);
                }
            o = make_ulonglong2(f64_canon(a0, qq.x, qq.y), f64_canon(a1, qq.x, qq.y));
        } else {
            Acc128 a0, a1;
#pragma unroll
            for (int i = 0; i < MAXA; ++i)
                if (i < (int)ns) {
                    const u64 w = __ldg(cv + (size_t)i * a.ne + s);
                    a0.mac(y[i][0], w);
                    a1.mac(y[i][1], w);
                }
            o = make_ulonglong2(a0.reduce(m), a1.reduce(m));
        }
        *reinterpret_cast<ulonglong2 *>(xo + ((size_t)s << log_n)) = o;
    }
}

// ---- FP64 fast base conversion core (every source and target prime FP64-mode) -------------
// out_t = sum_k y_k W[k][t] mod m_t for CONV_E consecutive coefficients per thread: the sources
// are exact doubles (< 2^42) held in registers, the weights W (doubles) and the targets' (q, 1/q)
// sit in shared memory (read as warp broadcasts), every term is an exact FMA two-product
// reduced to |r| < 2.5 m_t and summed in a double (< 2.5 17 m_t < 2^48).  One CTA = 128 threads
// x CONV_E coefficients of one group (digit or polynomial) and a chunk of <= CONV_TC targets.
// (Measured alternatives: 2 coefficients x 8 targets per thread, +4 %; Karatsuba-split products
// without per-term reduction -- 3 FMAs per term instead of 7 FP64 operations, 150 registers --
// +4 % / +20 %: the kernels are latency-, not FP64-issue-bound at these grid sizes.)
constexpr int CONV_E = 4, CONV_TC = 16, CONV_SRC = 17;

__device__ __forceinline__ void conv_fill_w(double *sW, int x, double w) { sW[x] = w; }
__device__ __forceinline__ void conv_fill_q(double2 *sQ, int j, double2 qq, u64) { sQ[j] = qq; }

template <int MAXS>
__device__ __forceinline__ void conv_f64_targets(const double (&yd)[MAXS][CONV_E], int ns, const double *sW,
                                                 const double2 *sQ, int tc, u64 *out, const u32 *sRow, u32 log_n)
{
    for (int j = 0; j < tc; ++j) {
        const double2 qq = sQ[j];
        double acc[CONV_E];
#pragma unroll
        for (int e = 0; e < CONV_E; ++e) acc[e] = 0.0;
#pragma unroll
        for (int k = 0; k < MAXS; ++k)
            if (k < ns) {
                const double w = sW[k * CONV_TC + j];
#pragma unroll
                for (int e = 0; e < CONV_E; ++e) acc[e] += f64_mac_term(yd[k][e], w, qq.x, qq.y);
            }
        u64 o[CONV_E];
#pragma unroll
        for (int e = 0; e < CONV_E; ++e) o[e] = f64_canon(acc[e], qq.x, qq.y);
        ulonglong2 *d = reinterpret_cast<ulonglong2 *>(out + ((size_t)sRow[j] << log_n));
#pragma unroll
        for (int h = 0; h < CONV_E / 2; ++h) d[h] = make_ulonglong2(o[2 * h], o[2 * h + 1]);
    }
}

// ModUp conversion, FP64 (k_modup_conv2's f64in case with every target slot FP64-mode):
// grid = (cnt * beta) x nchunks x N / (128 CONV_E); chunk = up to CONV_TC of the digit's target slots
template <int MAXA>
__global__ void __launch_bounds__(128) k_modup_conv_f64(ModUpConvArgs a, Tables tb, u32 nchunks)
{
    __shared__ double sW[CONV_SRC * CONV_TC];
    __shared__ double2 sQ[CONV_TC];
    __shared__ u32 sSlot[CONV_TC];
    const u32 log_n = tb.log_n;
    const u32 per_cd = (1u << log_n) / (128 * CONV_E);
    u32 b = blockIdx.x;
    const u32 cb = b % per_cd;
    b /= per_cd;
    const u32 sc = b % nchunks;
    b /= nchunks;
    const u32 d = b % a.beta, c = b / a.beta;
    const u32 lo = d * a.alpha, ns = min(a.alpha, a.l - lo);
    const u32 nt = a.ne - ns, t0 = sc * CONV_TC;
    if (t0 >= nt) return;  // (uniform per CTA) a full digit has fewer targets than the partial last one
    const u32 tc = min((u32)CONV_TC, nt - t0);
    if (threadIdx.x < tc) {  // list entry t0 + j -> slot (the digit's own slots are skipped)
        const u32 e = t0 + threadIdx.x, slot = e < lo ? e : e + ns;
        const u32 prime = slot < a.l ? slot : a.L + (slot - a.l);
        sSlot[threadIdx.x] = slot;
        conv_fill_q(sQ, threadIdx.x, __ldg(tb.psif + ((size_t)prime << log_n)), __ldg(&tb.mod[prime].q));
    }
    for (u32 x = threadIdx.x; x < ns * CONV_TC; x += 128) {
        const u32 k = x / CONV_TC, j = x % CONV_TC;
        if (j < tc) {
            const u32 e = t0 + j, slot = e < lo ? e : e + ns;
            conv_fill_w(sW, x, u2d(__ldg(a.conv + ((size_t)d * a.alpha + k) * a.ne + slot)));
        }
    }
    const u32 idx = cb * (128 * CONV_E) + CONV_E * threadIdx.x;
    double yd[MAXA][CONV_E];
#pragma unroll
    for (int k = 0; k < MAXA; ++k) {
#pragma unroll
        for (int e = 0; e < CONV_E; ++e) yd[k][e] = 0.0;
        if (k < (int)ns) {
            const ModC m = load_mod(tb.mod, lo + k);
            const ulonglong2 w = __ldg(a.yinv + (size_t)d * a.alpha + k);
            const ulonglong2 *xp = reinterpret_cast<const ulonglong2 *>(a.D + (((size_t)c * a.l + lo + k) << log_n) + idx);
#pragma unroll
            for (int h = 0; h < CONV_E / 2; ++h) {
                const ulonglong2 x = xp[h];
                yd[k][2 * h] = u2d(shoup(x.x, w.x, w.y, m.q));
                yd[k][2 * h + 1] = u2d(shoup(x.y, w.x, w.y, m.q));
            }
        }
    }
    __syncthreads();
    conv_f64_targets<MAXA>(yd, (int)ns, sW, sQ, (int)tc, a.X + (((size_t)c * a.beta + d) * a.ne << log_n) + idx, sSlot,
                           log_n);
}

// NTT tasks over the X slots that are not inside their own digit
struct TaskHybSlot {
    u64 *X;
    u32 l, L, alpha, beta, ne, log_n;
    u64 skip_mask = 0;  // slots (bit s) this launch leaves to the other arithmetic class
    int raw = 0;        // k_fwd_rows_store: FP64-mode slots hold lazy doubles (k_fwd_cols_r16)
    __device__ bool get(u32 r, const u64 *&s, u64 *&d, u32 &prime, u32 &sprime) const
    {
        const u32 slot = r % ne, dg = (r / ne) % beta;
        const u32 lo = dg * alpha, hi = min(lo + alpha, l);
        if (slot >= lo && slot < hi) return false;
        if (slot < 64 && ((skip_mask >> slot) & 1)) return false;
        d = X + ((size_t)r << log_n);
        s = d;
        prime = sprime = slot < l ? slot : L + (slot - l);
        return true;
    }
};

// acc_s = sum_d x~_{d,s} * key_{d, s}  (NTT form); x~ = din limb s inside its digit
struct FHybIP {
    static constexpr const char *NAME = "hyb_ip";
    static constexpr double MULS = 0, WORDS = 0;
    const u64 *X;   // [cnt][beta][ne][N] NTT form
    PolyMap din;    // NTT-form polynomial being switched (one poly per ciphertext)
    const u32 *perm;
    const u64 *key; // [dnum][2][L+K][N]
    u64 *ext;       // [cnt][2][ne][N]
    u32 l, L, K, alpha, beta, ne;
};

template <class Acc, int MAXB = 0>
__device__ __forceinline__ void hyb_ip_body(const FHybIP &a, const ModC &m, u32 log_n, u32 c, u32 s, u32 idx,
                                            u32 prime)
{
    const size_t n = (size_t)1 << log_n;
    const size_t LK = a.L + a.K;
    Acc b0, b1, c0, c1;  // (poly 0, poly 1) x (element idx, idx + 1)
    if constexpr (MAXB > 0) {  // every digit's operands in flight before the first multiply
        ulonglong2 x[MAXB], wb[MAXB], wa[MAXB];
#pragma unroll
        for (int d = 0; d < MAXB; ++d)
            if (d < (int)a.beta) {
                const u32 lo = d * a.alpha, hi = min(lo + a.alpha, a.l);
                if (s >= lo && s < hi) {
                    const u64 *dp = a.din.base + (((size_t)c * a.din.cap + s) << log_n);
                    x[d] = a.perm ? make_ulonglong2(dp[__ldg(a.perm + idx)], dp[__ldg(a.perm + idx + 1)])
                                  : *reinterpret_cast<const ulonglong2 *>(dp + idx);
                } else {
                    x[d] = *reinterpret_cast<const ulonglong2 *>(a.X + (((size_t)c * a.beta + d) * a.ne + s) * n + idx);
                }
                const ulonglong2 *kb =
                    reinterpret_cast<const ulonglong2 *>(a.key + (((size_t)2 * d) * LK + prime) * n + idx);
                wb[d] = __ldcs(kb);
                wa[d] = __ldcs(kb + LK * n / 2);
            }
#pragma unroll
        for (int d = 0; d < MAXB; ++d)
            if (d < (int)a.beta) {
                b0.mac(x[d].x, wb[d].x);
                b1.mac(x[d].y, wb[d].y);
                c0.mac(x[d].x, wa[d].x);
                c1.mac(x[d].y, wa[d].y);
            }
        u64 *e = a.ext + (((size_t)c * 2 * a.ne + s) << log_n) + idx;
        *reinterpret_cast<ulonglong2 *>(e) = make_ulonglong2(b0.reduce(m), b1.reduce(m));
        *reinterpret_cast<ulonglong2 *>(e + (size_t)a.ne * n) = make_ulonglong2(c0.reduce(m), c1.reduce(m));
    } else {
        for (u32 d = 0; d < a.beta; ++d) {
            const u32 lo = d * a.alpha, hi = min(lo + a.alpha, a.l);
            ulonglong2 x;
            if (s >= lo && s < hi) {
                const u64 *dp = a.din.base + (((size_t)c * a.din.cap + s) << log_n);
                x = a.perm ? make_ulonglong2(dp[__ldg(a.perm + idx)], dp[__ldg(a.perm + idx + 1)])
                           : *reinterpret_cast<const ulonglong2 *>(dp + idx);
            } else {
                x = *reinterpret_cast<const ulonglong2 *>(a.X + (((size_t)c * a.beta + d) * a.ne + s) * n + idx);
            }
            const ulonglong2 *kb = reinterpret_cast<const ulonglong2 *>(a.key + (((size_t)2 * d) * LK + prime) * n + idx);
            const ulonglong2 wb = __ldcs(kb), wa = __ldcs(kb + LK * n / 2);
            b0.mac(x.x, wb.x);
            b1.mac(x.y, wb.y);
            c0.mac(x.x, wa.x);
            c1.mac(x.y, wa.y);
        }
        u64 *e = a.ext + (((size_t)c * 2 * a.ne + s) << log_n) + idx;
        *reinterpret_cast<ulonglong2 *>(e) = make_ulonglong2(b0.reduce(m), b1.reduce(m));
        *reinterpret_cast<ulonglong2 *>(e + (size_t)a.ne * n) = make_ulonglong2(c0.reduce(m), c1.reduce(m));
    }
}

__global__ void __launch_bounds__(256) k_hyb_ip(FHybIP a, const ModC *mods, u32 log_n, u32 cnt)
{
    const size_t n = (size_t)1 << log_n;
    const size_t gid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (((size_t)cnt * a.ne * n) >> 1)) return;
    const u32 idx = (u32)((gid << 1) & (n - 1));
    const u32 s = (u32)(((gid << 1) >> log_n) % a.ne), c = (u32)(((gid << 1) >> log_n) / a.ne);
    const u32 prime = s < a.l ? s : a.L + (s - a.l);
    const ModC m = load_mod(mods, prime);
    if (a.beta <= 4) {
        if (m.q < (1ull << 40))
            hyb_ip_body<Acc40, 4>(a, m, log_n, c, s, idx, prime);
        else
            hyb_ip_body<Acc128, 4>(a, m, log_n, c, s, idx, prime);
    } else if (m.q < (1ull << 40))
        hyb_ip_body<Acc40>(a, m, log_n, c, s, idx, prime);
    else
        hyb_ip_body<Acc128>(a, m, log_n, c, s, idx, prime);
}

// Y[p][i] = conv_{P}(acc_p restricted to the special slots) mod q_i, i < l  (coefficient form)
struct ModDownConvArgs {
    const u64 *ext;  // [npolys][ne][N], special slots l..l+K-1 in coefficient form
    u64 *Y;          // [npolys][l][N]
    const ulonglong2 *pyinv;  // [K] (P/p_k)^{-1} mod p_k
    const u64 *conv;          // [K][L] (P/p_k) mod q_i
    u32 l, L, K, ne;
};

__global__ void __launch_bounds__(128) k_moddown_conv(ModDownConvArgs a, const ModC *mods, u32 log_n, u32 npolys)
{
    const size_t n = (size_t)1 << log_n;
    const size_t gid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (((size_t)npolys * n) >> 1)) return;
    const u32 idx = (u32)((gid << 1) & (n - 1)), p = (u32)((gid << 1) >> log_n);
    u64 y[HYB_MAX_ALPHA][2];
#pragma unroll
    for (int k = 0; k < HYB_MAX_ALPHA; ++k)
        if (k < (int)a.K) {
            const ModC m = load_mod(mods, a.L + k);
            const ulonglong2 w = __ldg(a.pyinv + k);
            const ulonglong2 x =
                *reinterpret_cast<const ulonglong2 *>(a.ext + (((size_t)p * a.ne + a.l + k) << log_n) + idx);
            y[k][0] = shoup(x.x, w.x, w.y, m.q);
            y[k][1] = shoup(x.y, w.x, w.y, m.q);
        }
    u64 *yo = a.Y + (((size_t)p * a.l) << log_n) + idx;
    for (u32 i = 0; i < a.l; ++i) {
        const ModC m = load_mod(mods, i);
        u64 o0, o1;
        conv_slot<Acc128>(y, a.K, a.conv + i, a.L, m, o0, o1);
        *reinterpret_cast<ulonglong2 *>(yo + (size_t)i * n) = make_ulonglong2(o0, o1);
    }
}

// ModDown conversion v2: targets split into chunks over gridDim (the v1 kernel looped over
// all l targets per thread: 512 CTAs at N = 2^16, latency-bound), K-specialised registers.
template <int MAXK>
__global__ void __launch_bounds__(128) k_moddown_conv2(ModDownConvArgs a, const ModC *mods, u32 log_n, u32 nchunks,
                                                       u32 chunk)
{
    const u32 n = 1u << log_n, per_p = n >> 8;
    u32 b = blockIdx.x;
    const u32 cb = b % per_p;
    b /= per_p;
    const u32 sc = b % nchunks, p = b / nchunks;
    const u32 idx = (cb << 8) + 2 * threadIdx.x;
    u64 y[MAXK][2];
#pragma unroll
    for (int k = 0; k < MAXK; ++k) {
        y[k][0] = y[k][1] = 0;
        if (k < (int)a.K) {
            const ModC m = load_mod(mods, a.L + k);
            const ulonglong2 w = __ldg(a.pyinv + k);
            const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(a.ext + (((size_t)p * a.ne + a.l + k) << log_n) + idx);
            y[k][0] = shoup(x.x, w.x, w.y, m.q);
            y[k][1] = shoup(x.y, w.x, w.y, m.q);
        }
    }
    u64 *yo = a.Y + (((size_t)p * a.l) << log_n) + idx;
    const u32 i1 = min(a.l, (sc + 1) * chunk);
    for (u32 i = sc * chunk; i < i1; ++i) {
        const ModC m = load_mod(mods, i);
        Acc128 a0, a1;
#pragma unroll
        for (int k = 0; k < MAXK; ++k)
            if (k < (int)a.K) {
                const u64 w = __ldg(a.conv + (size_t)k * a.L + i);
                a0.mac(y[k][0], w);
                a1.mac(y[k][1], w);
            }
        *reinterpret_cast<ulonglong2 *>(yo + ((size_t)i << log_n)) = make_ulonglong2(a0.reduce(m), a1.reduce(m));
    }
}

template <int B1, int B2>
void hyb_ntt_impl(const Launch &L, const TaskHybSlot &t, u32 nslots, bool cols_only = false)
{
    const u32 g1 = (1u << B2) / COLS;
    const double nh = (double)nslots * (1u << (B1 + B2 - 1)), nb = (double)nslots * (8u << (B1 + B2));
    double fw = 0, wt = 0;  // slots weighted by the digits that convert into them
    for (u32 dg = 0; dg < t.beta; ++dg)
        for (u32 slot = 0; slot < t.ne; ++slot) {
            const u32 lo = dg * t.alpha, hi = std::min(lo + t.alpha, t.l);
            if (slot >= lo && slot < hi) continue;
            fw += f64_prime(L, slot < t.l ? slot : t.L + (slot - t.l)) ? 1 : 0;
            wt += 1;
        }
    const double f = wt > 0 ? fw / wt : 0;
    TaskHybSlot tr = t;
    if (B1 >= 6 && fw > 0 && t.ne <= 64) {  // FP64 slots: radix-16 columns (lazy doubles); the rest generic
        u64 fmask = 0;
        for (u32 slot = 0; slot < t.ne; ++slot)
            if (f64_prime(L, slot < t.l ? slot : t.L + (slot - t.l))) fmask |= 1ull << slot;
        TaskHybSlot tf = t;
        tf.skip_mask = ~fmask;
        const double ff = nh * (fw / wt);
        KLAUNCH(L, "hyb_ntt_cols", nttw(ff * B1, 1.0, 0, 2 * nb * (fw / wt)),
                (k_fwd_cols_r16<(B1 >= 6 ? B1 : 6), B2, TaskHybSlot><<<nslots * g1, 1 << B1, 0, L.st>>>(tf, *L.tb, g1)));
        if (fw < wt) {
            TaskHybSlot ti = t;
            ti.skip_mask = fmask;
            KLAUNCH(L, "hyb_ntt_cols", nttw((nh - ff) * B1, 0.0, 0, 2 * nb * (1 - fw / wt)),
                    (k_fwd_cols<B1, B2, TaskHybSlot><<<nslots * g1, COLS * (1 << B1) / 8, 0, L.st>>>(ti, *L.tb, g1)));
        }
        tr.raw = 1;
    } else {
        KLAUNCH(L, "hyb_ntt_cols", nttw(nh * B1, f, 0, 2 * nb),
                (k_fwd_cols<B1, B2, TaskHybSlot><<<nslots * g1, COLS * (1 << B1) / 8, 0, L.st>>>(t, *L.tb, g1)));
    }
    if (cols_only) return;  // the inner product (k_ks_mac hybrid mode) applies the row phase
    const u32 g2 = (1u << B1) / RowGeom<B2>::R;
    KLAUNCH(L, "hyb_ntt_rows", nttw(nh * B2, f, 0, 2 * nb),
            (k_fwd_rows_store<B2, TaskHybSlot><<<nslots * g2, 128, 0, L.st>>>(tr, *L.tb, g2)));
}

template <int B1, int B2>
void cols_submul_impl(const Launch &L, const TaskPlainCol &t, const SubMulArgs &a, u32 nlimbs)
{
    const u32 g1 = (1u << B2) / COLS;
    const double nh = (double)nlimbs * (1u << (B1 + B2 - 1)), nb = (double)nlimbs * (8u << (B1 + B2));
    const double f = f64_share(L, t.ls);
    SubMulArgs as = a;
    if (f == 1.0 && B1 >= 6) {  // every limb FP64-mode: radix-16 columns, lazy-double rows
        KLAUNCH(L, "ntt_fwd_cols", nttw(nh * B1, f, 0, 2 * nb),
                (k_fwd_cols_r16<(B1 >= 6 ? B1 : 6), B2, TaskPlainCol><<<nlimbs * g1, 1 << B1, 0, L.st>>>(t, *L.tb, g1)));
        as.s_raw = 1;
    } else {
        KLAUNCH(L, "ntt_fwd_cols", nttw(nh * B1, f, 0, 2 * nb),
                (k_fwd_cols<B1, B2, TaskPlainCol><<<nlimbs * g1, COLS * (1 << B1) / 8, 0, L.st>>>(t, *L.tb, g1)));
    }
    const u32 g2 = (1u << B1) / RowGeom<B2>::R;
    KLAUNCH(L, "submul_rows", nttw(nh * B2, f, 2 * nh, (a.base.base ? 4 : 3) * nb),
            (k_fwd_rows_submul<B2><<<nlimbs * g2, 128, 0, L.st>>>(as, *L.tb, g2)));
}
}  // namespace

// every extended slot FP64-mode (q_i and the special primes < 2^42) at N >= 2^12 with ne <= 64:
// ModUp leaves the column phase's lazy doubles and the inner product continues with the row phase
bool hyb_fused_ip_ok(const Launch &L, u32 l, u32 Lq, u32 K)
{
    const char *e = std::getenv("CKKS_HYB_FUSED_IP");  // =0: separate row-phase and inner-product launches (A/B)
    if (L.tb->log_n < 12 || l + K > 64) return false;
    if (L.key_compact) return true;  // compact key rows (every limb < 2^40): only k_ks_mac reads them
    if (e && e[0] == '0') return false;
    for (u32 i = 0; i < l; ++i)
        if (!f64_prime(L, i)) return false;
    for (u32 k = 0; k < K; ++k)
        if (!f64_prime(L, Lq + k)) return false;
    return true;
}

void launch_hyb_ip_fused(const Launch &L, const u64 *X, PolyMap din, const u32 *perm, const u64 *key, u64 *ext, u32 cnt,
                         u32 l, u32 Lq, u32 K, u32 alpha, u32 beta, u32 ne, PolyMap zbase, const ulonglong2 *zrs)
{
    MacArgs a{};
    if (zrs) {
        a.rs_rows = 1;
        a.zbase = zbase;
        a.zrs = zrs;
    }
    a.I = X;
    a.din = din;
    a.perm = perm;
    a.key = key;
    a.ext = ext;
    a.Lk = Lq;
    a.l = l;
    a.t0 = 0;
    a.T = ne;
    a.sp = Lq;
    a.t0i = 0;
    a.Ti = ne;
    a.halpha = alpha;
    a.nd = beta;
    a.next = ne;
    a.kst = Lq + K;
#define CALLM(b1, b2) mac_launch<b2>(L, a, cnt * ne, 5)
    CKKS_DISPATCH_LOGN(L.tb->log_n, CALLM)
#undef CALLM
}

void launch_hyb_modup(const Launch &L, const u64 *D, u64 *X, const ulonglong2 *yinv, const u64 *conv, u32 cnt, u32 l,
                      u32 Lq, u32 K, u32 alpha, u32 beta, u32 ne, bool cols_only)
{
    ModUpConvArgs a{D, X, yinv, conv, l, Lq, K, alpha, beta, ne};
    const size_t total = ((size_t)cnt * beta) << L.tb->log_n;
    const double conv_macs = (double)total * ((double)ne - (double)alpha) * alpha;
    const char *ce = std::getenv("CKKS_MODUP_CONV");
    if (ce && ce[0] == '1') {  // v1: generic integer accumulators (kept for A/B and tests)
        KLAUNCH(L, "hyb_modup_conv", (Work{0, conv_macs + (double)total * alpha, 8.0 * (double)total * (alpha + ne)}),
                (k_modup_conv<<<(unsigned)((total / 2 * ((ne + CONV_SLOTS - 1) / CONV_SLOTS) + 127) / 128), 128, 0,
                                 L.st>>>(a, L.tb->mod, L.tb->log_n, cnt)));
    } else {
        bool f64in = true;  // every digit prime FP64-mode: residues fit the FP64 two-product
        for (u32 i = 0; i < l; ++i) f64in = f64in && f64_prime(L, i);
        u32 nf64 = 0;
        for (u32 sl = 0; sl < ne; ++sl) nf64 += f64_prime(L, sl < l ? sl : Lq + (sl - l)) ? 1 : 0;
        if (f64in && nf64 == ne && (L.tb->log_n >= 9) && !std::getenv("CKKS_CONV_V2")) {
            const u32 nt_max = ne - (l - (beta - 1) * alpha), nchunks = (nt_max + CONV_TC - 1) / CONV_TC;
            const unsigned blocks = (unsigned)((size_t)cnt * beta * nchunks * ((1u << L.tb->log_n) / (128 * CONV_E)));
            const Work w{0, (double)total * alpha, 8.0 * (double)total * (alpha + ne), 0, conv_macs};
#define CONV3(A) KLAUNCH(L, "hyb_modup_conv", w, (k_modup_conv_f64<A><<<blocks, 128, 0, L.st>>>(a, *L.tb, nchunks)))
            if (alpha <= 4) CONV3(4);
            else if (alpha <= 8) CONV3(8);
            else if (alpha <= 10) CONV3(10);
            else if (alpha <= 12) CONV3(12);
            else CONV3(16);
#undef CONV3
            TaskHybSlot t{X, l, Lq, alpha, beta, ne, L.tb->log_n};
#define CALLH(b1, b2) hyb_ntt_impl<b1, b2>(L, t, cnt * beta * ne, cols_only)
            CKKS_DISPATCH_LOGN(L.tb->log_n, CALLH)
#undef CALLH
            return;
        }
        const char *che = std::getenv("CKKS_CONV_CHUNK");
        const u32 chunk = che ? (u32)std::max(1, std::atoi(che)) : 16, nchunks = (ne + chunk - 1) / chunk;
        const unsigned blocks = (unsigned)((size_t)cnt * beta * nchunks * (L.tb->log_n >= 8 ? (1u << (L.tb->log_n - 8)) : 1));
        const double fmac = f64in ? (double)total * alpha * nf64 : 0;
        const Work w{0, conv_macs - fmac + (double)total * alpha, 8.0 * (double)total * (alpha + ne), 0, fmac};
#define CONV2(A) KLAUNCH(L, "hyb_modup_conv", w, (k_modup_conv2<A><<<blocks, 128, 0, L.st>>>(a, *L.tb, nchunks, chunk, f64in)))
        if (alpha <= 2) CONV2(2);
        else if (alpha <= 4) CONV2(4);
        else if (alpha <= 6) CONV2(6);
        else if (alpha <= 8) CONV2(8);
        else if (alpha <= 10) CONV2(10);
        else if (alpha <= 12) CONV2(12);
        else CONV2(16);
#undef CONV2
    }
    TaskHybSlot t{X, l, Lq, alpha, beta, ne, L.tb->log_n};
#define CALLH(b1, b2) hyb_ntt_impl<b1, b2>(L, t, cnt * beta * ne, cols_only)
    CKKS_DISPATCH_LOGN(L.tb->log_n, CALLH)
#undef CALLH
}

void launch_hyb_ip(const Launch &L, const u64 *X, PolyMap din, const u32 *perm, const u64 *key, u64 *ext, u32 cnt,
                   u32 l, u32 Lq, u32 K, u32 alpha, u32 beta, u32 ne)
{
    FHybIP a{X, din, perm, key, ext, l, Lq, K, alpha, beta, ne};
    const size_t total = ((size_t)cnt * ne) << L.tb->log_n;
    KLAUNCH(L, "hyb_ip", (Work{0, 2.0 * (double)total * beta, 8.0 * (double)total * (3.0 * beta + 2)}),
            (k_hyb_ip<<<(unsigned)((total / 2 + 255) / 256), 256, 0, L.st>>>(a, L.tb->mod, L.tb->log_n, cnt)));
}

void launch_hyb_moddown(const Launch &L, u64 *ext, u64 *Y, const ulonglong2 *pyinv, const u64 *conv, u32 npolys, u32 l,
                        u32 Lq, u32 K, u32 ne, PolyMap out, PolyMap base, const u32 *base_perm, bool base_c0_only,
                        const ulonglong2 *pinv, PolyMap acc)
{
    // INTT of the K special slots (both polynomials of every ciphertext)
    launch_ntt_inv(L, PolyMap{ext + ((size_t)l << L.tb->log_n), ne}, PolyMap{ext + ((size_t)l << L.tb->log_n), ne},
                   npolys, LimbSet{K, 0, 0, Lq}, nullptr);
    ModDownConvArgs a{ext, Y, pyinv, conv, l, Lq, K, ne};
    const size_t total = (size_t)npolys << L.tb->log_n;
    const Work w{0, (double)total * K * (l + 1), 8.0 * (double)total * (K + l)};
    const char *ce = std::getenv("CKKS_MODDOWN_CONV");
    if (ce && ce[0] == '1') {
        KLAUNCH(L, "hyb_moddown_conv", w,
                (k_moddown_conv<<<(unsigned)((total / 2 + 127) / 128), 128, 0, L.st>>>(a, L.tb->mod, L.tb->log_n, npolys)));
    } else {
        const u32 chunk = 8, nchunks = (l + chunk - 1) / chunk;
        const unsigned blocks = (unsigned)((size_t)npolys * nchunks * (L.tb->log_n >= 8 ? (1u << (L.tb->log_n - 8)) : 1));
#define MDC2(K_) KLAUNCH(L, "hyb_moddown_conv", w, (k_moddown_conv2<K_><<<blocks, 128, 0, L.st>>>(a, L.tb->mod, L.tb->log_n, nchunks, chunk)))
        if (K <= 2) MDC2(2);
        else if (K <= 4) MDC2(4);
        else if (K <= 8) MDC2(8);
        else MDC2(16);
#undef MDC2
    }
    TaskPlainCol t{PolyMap{Y, l}, PolyMap{Y, l}, LimbSet{l, l, 0, Lq}, L.tb->log_n, make_fdiv(l)};
    SubMulArgs s{Y, l, 0, PolyMap{ext, ne}, out, base, acc, base_perm, base_c0_only ? 1 : 0, pinv};
#define CALLS(b1, b2) cols_submul_impl<b1, b2>(L, t, s, npolys * l)
    CKKS_DISPATCH_LOGN(L.tb->log_n, CALLS)
#undef CALLS
}

namespace {
// ---- fused hybrid ModDown + RESCALE (internal.h launch_hyb_moddown_rs) ----------------------
struct HybRsArgs {
    u64 *ext;                 // [npolys][ne][N]
    PolyMap base;             // tensor (d0, d1)
    u64 *W;                   // [npolys][l-1][N]
    const ulonglong2 *pyinv;  // [K] (P/p_k)^{-1} mod p_k
    const u64 *conv;          // [K][L] (P/p_k) mod q_i
    const ulonglong2 *rs;     // [3][l]
    u32 l, L, K, ne;
};

// ext slot l-1 <- P base_{l-1} + acc_{l-1} mod q_{l-1} (NTT form; its INTT is the U of the fused tail)
__global__ void __launch_bounds__(256) k_hyb_rs_z(HybRsArgs a, const ModC *mods, u32 log_n, u32 npolys)
{
    const size_t n = (size_t)1 << log_n;
    const size_t gid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= ((size_t)npolys * n) >> 1) return;
    const u32 idx = (u32)((gid << 1) & (n - 1)), p = (u32)((gid << 1) >> log_n);
    const u32 il = a.l - 1;
    const ModC m = load_mod(mods, il);
    const ulonglong2 pm = __ldg(a.rs + il);
    u64 *e = a.ext + (((size_t)p * a.ne + il) << log_n) + idx;
    const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(e);
    const ulonglong2 d = *reinterpret_cast<const ulonglong2 *>(limb_ptr(a.base, p, il, log_n) + idx);
    *reinterpret_cast<ulonglong2 *>(e) =
        make_ulonglong2(addmod(shoup(d.x, pm.x, pm.y, m.q), x.x, m.q), addmod(shoup(d.y, pm.x, pm.y, m.q), x.y, m.q));
}

// W_i = Y_i + [P]_{q_i} g (coefficient form), Y = conv_P(acc restricted to the special slots),
// g = (U - Y_{l-1}) P^{-1} mod q_{l-1}; one thread = 2 coefficients of one polynomial and a chunk of
// targets.  FP64-mode specials and targets (every prime < 2^42) accumulate on the FP64 pipe
// (exact two-product terms, |term| < 2.5 q_i, K + 1 <= 17 of them), 60-bit specials in 128 bits.
template <int MAXK>
__global__ void __launch_bounds__(128) k_hyb_rs_conv(HybRsArgs a, Tables tb, u32 nchunks, u32 chunk, int f64)
{
    const u32 log_n = tb.log_n;
    const u32 n = 1u << log_n, per_p = n >> 8;
    u32 b = blockIdx.x;
    const u32 cb = b % per_p;
    b /= per_p;
    const u32 sc = b % nchunks, p = b / nchunks;
    const u32 idx = (cb << 8) + 2 * threadIdx.x;
    const u64 *ep = a.ext + (((size_t)p * a.ne) << log_n) + idx;
    u64 y[MAXK][2];
#pragma unroll
    for (int k = 0; k < MAXK; ++k) {
        y[k][0] = y[k][1] = 0;
        if (k < (int)a.K) {
            const ModC m = load_mod(tb.mod, a.L + k);
            const ulonglong2 w = __ldg(a.pyinv + k);
            const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(ep + ((size_t)(a.l + k) << log_n));
            y[k][0] = shoup(x.x, w.x, w.y, m.q);
            y[k][1] = shoup(x.y, w.x, w.y, m.q);
        }
    }
    const u32 il = a.l - 1;
    u64 g0, g1;
    {  // g = (U - Y_{l-1}) P^{-1} mod q_{l-1}, canonical (the rescale's [h_{l-1}]_{q_{l-1}})
        const ModC m = load_mod(tb.mod, il);
        Acc128 s0, s1;
#pragma unroll
        for (int k = 0; k < MAXK; ++k)
            if (k < (int)a.K) {
                const u64 w = __ldg(a.conv + (size_t)k * a.L + il);
                s0.mac(y[k][0], w);
                s1.mac(y[k][1], w);
            }
        const ulonglong2 u = *reinterpret_cast<const ulonglong2 *>(ep + ((size_t)il << log_n));
        const ulonglong2 pinv = __ldg(a.rs + a.l + il);
        g0 = shoup(u.x + m.q - s0.reduce(m), pinv.x, pinv.y, m.q);
        g1 = shoup(u.y + m.q - s1.reduce(m), pinv.x, pinv.y, m.q);
    }
    u64 *wo = a.W + (((size_t)p * il) << log_n) + idx;
    const u32 i1 = min(il, (sc + 1) * chunk);
    for (u32 i = sc * chunk; i < i1; ++i) {
        const ModC m = load_mod(tb.mod, i);
        const u64 pm = __ldg(&a.rs[2 * a.l + i].x);
        ulonglong2 o;
        if (f64 && m.q < tb.f64_qmax) {
            const double2 qq = __ldg(tb.psif + ((size_t)i << log_n));  // entry 0: (q, 1/q)
            const double pmd = u2d(pm);
            double a0 = f64_mac_term(u2d(g0), pmd, qq.x, qq.y), a1 = f64_mac_term(u2d(g1), pmd, qq.x, qq.y);
#pragma unroll
            for (int k = 0; k < MAXK; ++k)
                if (k < (int)a.K) {
                    const double w = u2d(__ldg(a.conv + (size_t)k * a.L + i));
                    a0 += f64_mac_term(u2d(y[k][0]), w, qq.x, qq.y);
                    a1 += f64_mac_term(u2d(y[k][1]), w, qq.x, qq.y);
                }
            o = make_ulonglong2(f64_canon(a0, qq.x, qq.y), f64_canon(a1, qq.x, qq.y));
        } else {
            Acc128 a0, a1;
            a0.mac(g0, pm);
            a1.mac(g1, pm);
#pragma unroll
            for (int k = 0; k < MAXK; ++k)
                if (k < (int)a.K) {
                    const u64 w = __ldg(a.conv + (size_t)k * a.L + i);
                    a0.mac(y[k][0], w);
                    a1.mac(y[k][1], w);
                }
            o = make_ulonglong2(a0.reduce(m), a1.reduce(m));
        }
        *reinterpret_cast<ulonglong2 *>(wo + ((size_t)i << log_n)) = o;
    }
}

// FP64 version of k_hyb_rs_conv (every special prime and q_0..q_{l-1} FP64-mode): the sources are
// y_0..y_{K-1} and g (weight [P]_{q_i}), CONV_E coefficients per thread, weights in shared memory.
template <int MAXS>
__global__ void __launch_bounds__(128) k_hyb_rs_conv_f64(HybRsArgs a, Tables tb, u32 nchunks)
{
    __shared__ double sW[CONV_SRC * CONV_TC];
    __shared__ double2 sQ[CONV_TC];
    const u32 log_n = tb.log_n;
    const u32 per_p = (1u << log_n) / (128 * CONV_E);
    u32 b = blockIdx.x;
    const u32 cb = b % per_p;
    b /= per_p;
    const u32 sc = b % nchunks, p = b / nchunks;
    const u32 il = a.l - 1, t0 = sc * CONV_TC, tc = min((u32)CONV_TC, il - t0);
    const u32 K = a.K;
    __shared__ u32 sRow[CONV_TC];
    if (threadIdx.x < tc) {
        conv_fill_q(sQ, threadIdx.x, __ldg(tb.psif + ((size_t)(t0 + threadIdx.x) << log_n)),
                    __ldg(&tb.mod[t0 + threadIdx.x].q));
        sRow[threadIdx.x] = t0 + threadIdx.x;
    }
    for (u32 x = threadIdx.x; x < (K + 1) * CONV_TC; x += 128) {
        const u32 k = x / CONV_TC, j = x % CONV_TC;
        if (j < tc)
            conv_fill_w(sW, x, u2d(k < K ? __ldg(a.conv + (size_t)k * a.L + t0 + j) : __ldg(&a.rs[2 * a.l + t0 + j].x)));
    }
    const u32 idx = cb * (128 * CONV_E) + CONV_E * threadIdx.x;
    const u64 *ep = a.ext + (((size_t)p * a.ne) << log_n) + idx;
    double yd[MAXS][CONV_E];
#pragma unroll
    for (int k = 0; k < MAXS; ++k) {
#pragma unroll
        for (int e = 0; e < CONV_E; ++e) yd[k][e] = 0.0;
        if (k < (int)K) {
            const ModC m = load_mod(tb.mod, a.L + k);
            const ulonglong2 w = __ldg(a.pyinv + k);
            const ulonglong2 *xp = reinterpret_cast<const ulonglong2 *>(ep + ((size_t)(a.l + k) << log_n));
#pragma unroll
            for (int h = 0; h < CONV_E / 2; ++h) {
                const ulonglong2 x = xp[h];
                yd[k][2 * h] = u2d(shoup(x.x, w.x, w.y, m.q));
                yd[k][2 * h + 1] = u2d(shoup(x.y, w.x, w.y, m.q));
            }
        }
    }
    {  // g = (U - Y_{l-1}) P^{-1} mod q_{l-1}, canonical; source K
        const ModC m = load_mod(tb.mod, il);
        const double2 qq = __ldg(tb.psif + ((size_t)il << log_n));
        double acc[CONV_E];
#pragma unroll
        for (int e = 0; e < CONV_E; ++e) acc[e] = 0.0;
#pragma unroll
        for (int k = 0; k < MAXS - 1; ++k)
            if (k < (int)K) {
                const double w = u2d(__ldg(a.conv + (size_t)k * a.L + il));
#pragma unroll
                for (int e = 0; e < CONV_E; ++e) acc[e] += f64_mac_term(yd[k][e], w, qq.x, qq.y);
            }
        const ulonglong2 *up = reinterpret_cast<const ulonglong2 *>(ep + ((size_t)il << log_n));
        u64 u[CONV_E];
#pragma unroll
        for (int h = 0; h < CONV_E / 2; ++h) {
            const ulonglong2 x = up[h];
            u[2 * h] = x.x;
            u[2 * h + 1] = x.y;
        }
        const ulonglong2 pinv = __ldg(a.rs + a.l + il);
#pragma unroll
        for (int e = 0; e < CONV_E; ++e) {
            const u64 g = shoup(u[e] + m.q - f64_canon(acc[e], qq.x, qq.y), pinv.x, pinv.y, m.q);
#pragma unroll
            for (int k = 0; k < MAXS; ++k)
                if (k == (int)K) yd[k][e] = u2d(g);
        }
    }
    __syncthreads();
    conv_f64_targets<MAXS>(yd, (int)K + 1, sW, sQ, (int)tc, a.W + (((size_t)p * il) << log_n) + idx, sRow, log_n);
}
}  // namespace

void launch_hyb_moddown_rs(const Launch &L, u64 *ext, u64 *Y, const ulonglong2 *pyinv, const u64 *conv, u32 npolys,
                           u32 l, u32 Lq, u32 K, u32 ne, PolyMap out, PolyMap base, const ulonglong2 *rs,
                           bool rows_done)
{
    const u32 log_n = L.tb->log_n;
    const size_t total = (size_t)npolys << log_n;
    HybRsArgs a{ext, base, Y, pyinv, conv, rs, l, Lq, K, ne};
    // INTT of slot l-1 (U) and the K special slots: contiguous in ext
    const PolyMap tail{ext + ((size_t)(l - 1) << log_n), ne};
    if (rows_done) {  // z and the row phase applied by the inner product (MacArgs::rs_rows)
        launch_ntt_inv_cols(L, tail, npolys, LimbSet{K + 1, 1, l - 1, Lq});
    } else {
        KLAUNCH(L, "hyb_rs_z", (Work{0, (double)total, 8.0 * 3 * (double)total}),
                (k_hyb_rs_z<<<(unsigned)((total / 2 + 255) / 256), 256, 0, L.st>>>(a, L.tb->mod, log_n, npolys)));
        launch_ntt_inv(L, tail, tail, npolys, LimbSet{K + 1, 1, l - 1, Lq}, nullptr);
    }
    bool f64 = true;  // every special prime FP64-mode: the y_k fit the FP64 two-product
    for (u32 k = 0; k < K; ++k) f64 = f64 && f64_prime(L, Lq + k);
    bool f64q = true;
    for (u32 i = 0; i < l; ++i) f64q = f64q && f64_prime(L, i);
    if (f64 && f64q && log_n >= 9 && K + 1 <= (u32)CONV_SRC && !std::getenv("CKKS_CONV_V2")) {
        const u32 nchunks = (l - 1 + CONV_TC - 1) / CONV_TC;
        const unsigned blocks = (unsigned)((size_t)npolys * nchunks * ((1u << log_n) / (128 * CONV_E)));
        const double macs = (double)total * (K + 1) * (l - 1) + (double)total * K * nchunks;
        const Work w{0, (double)total * K, 8.0 * (double)total * (K + l), 0, macs};
#define RSF(S_) KLAUNCH(L, "hyb_moddown_conv", w, (k_hyb_rs_conv_f64<S_><<<blocks, 128, 0, L.st>>>(a, *L.tb, nchunks)))
        if (K + 1 <= 5) RSF(5);
        else if (K + 1 <= 9) RSF(9);
        else if (K + 1 <= 11) RSF(11);
        else if (K + 1 <= 13) RSF(13);
        else RSF(17);
#undef RSF
    } else {
    const u32 chunk = 8, nchunks = (l - 1 + chunk - 1) / chunk;
    const unsigned blocks = (unsigned)((size_t)npolys * nchunks * (log_n >= 8 ? (1u << (log_n - 8)) : 1));
    const double macs = (double)total * (K + 1) * (l - 1) + (double)total * K * nchunks;
    const Work w{0, f64 ? 0.0 : macs, 8.0 * (double)total * (K + l), 0, f64 ? macs : 0.0};
#define RSC(K_) KLAUNCH(L, "hyb_moddown_conv", w, (k_hyb_rs_conv<K_><<<blocks, 128, 0, L.st>>>(a, *L.tb, nchunks, chunk, f64 ? 1 : 0)))
    if (K <= 2) RSC(2);
    else if (K <= 4) RSC(4);
    else if (K <= 8) RSC(8);
    else RSC(16);
#undef RSC
    }
    TaskPlainCol t{PolyMap{Y, l - 1}, PolyMap{Y, l - 1}, LimbSet{l - 1, l - 1, 0, Lq}, log_n, make_fdiv(l - 1)};
    SubMulArgs s{Y, l - 1, 0, PolyMap{ext, ne}, out, base, PolyMap{nullptr, 0}, nullptr, 0, rs};
    s.bconsts = rs + l;
#define CALLS(b1, b2) cols_submul_impl<b1, b2>(L, t, s, npolys * (l - 1))
    CKKS_DISPATCH_LOGN(log_n, CALLS)
#undef CALLS
}

void launch_sum_strided(const Launch &L, PolyMap g, PolyMap out, u32 nout_ct, u32 np, u32 l, u32 R, u32 rs, u32 qs)
{
    run_elem(L, FSumStrided{g, out, R, rs, qs, np}, nout_ct * np, l);
}

// ---- fused ModDown + rescale helpers (reading A7: floor(floor(x / P) / q) = floor(x / (P q))) --
// z[p] = P d[p][l-1] + acc[p][l-1]  mod q_{l-1}   (NTT form, per coefficient)

namespace {
// ---- fused ModDown + rescale tail in two launches (reading A7) ---------------------------------
// k_fr_rows: the inverse row phase of z = P d_{l-1} + acc_{l-1} mod q_{l-1} (computed in the load;
// item 0) and of the special-prime accumulator acc_P (in place; item 1), per polynomial.
// k_fr_cols: both column phases in one CTA, then T = (acc_P - z) q_{l-1}^{-1} mod P straight from
// registers; z (coefficient form) and T are what the broadcast reads.  Replaces fr_z, two INTT
// launch pairs and fr_t (six launches of a few CTAs each).
struct FrTail {
    const u64 *d;  // tensor output (d0, d1), limb l-1 read
    u32 d_cap;
    u64 *acc;      // key-switch accumulators [np][acc_cap][N]: limb l-1 read, limb P (index acc_cap-1)
    u32 acc_cap;   //   receives its row phase in place
    u64 *z;        // [np][N]
    u64 *T;        // [np][N]
    u32 lm1, sp;   // prime indices of q_{l-1} and P
    ulonglong2 pm;    // P mod q_{l-1} (Shoup)
    ulonglong2 qinv;  // q_{l-1}^{-1} mod P (Shoup)
};

template <int B2>
__global__ void __launch_bounds__(128) k_fr_rows(FrTail a, Tables tb, u32 ngroups)
{
    using G = RowGeom<B2>;
    __shared__ u64 sm[G::R * G::SROW];
    const u32 log_n = tb.log_n;
    const u32 B1 = log_n - B2;
    const u32 r = blockIdx.x >> (31 - __clz(ngroups)), grp = blockIdx.x & (ngroups - 1);  // r = 2 p + item
    const u32 p = r >> 1, item = r & 1;
    const int rin = threadIdx.x / G::THR, lt = threadIdx.x % G::THR;
    const u32 row = grp * G::R + rin;
    const u32 prime = item ? a.sp : a.lm1;
    const ModC m = load_mod(tb.mod, prime);
    const u32 roff = row << B2;
    const size_t n = (size_t)1 << log_n;
    u64 *accp = a.acc + ((size_t)p * a.acc_cap + (item ? a.acc_cap - 1 : a.lm1)) * n + roff;
    u64 v[8];
    if (item) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = accp[(k << (B2 - 3)) | lt];
    } else {
        const u64 *dp = a.d + ((size_t)p * a.d_cap + a.lm1) * n + roff;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int e = (k << (B2 - 3)) | lt;
            v[k] = addmod(shoup(dp[e], a.pm.x, a.pm.y, m.q), accp[e], m.q);
        }
    }
    const RowEx ex{sm + rin * G::SROW};
    ex(v, lt, B2 - 3, 0);
    inv_rounds<B2, 0>(v, ex, lt, B1, row, tb.ipsi + ((size_t)prime << log_n), m.q, 0,
                      tb.ipsif + ((size_t)prime << log_n), use_f64(tb, m.q));
    u64 *drow = item ? accp : a.z + (size_t)p * n + roff;
#pragma unroll
    for (int i = 0; i < 8; ++i) drow[(i << (B2 - 3)) | lt] = v[i];
}

// (4 columns per CTA: the tail runs on 2 polynomials of one ciphertext, so more, smaller CTAs)
constexpr int FR_COLS = 4;
template <int B1, int B2>
__global__ void __launch_bounds__(2 * FR_COLS * (1 << B1) / 8) k_fr_cols(FrTail a, Tables tb, u32 ngroups)
{
    // threads [0, H): z's column phase (q_{l-1}); [H, 2H): acc_P's (P) -- the two transforms run
    // side by side (the P limb's 60-bit integer INTT was the kernel's serial latency), then the
    // P half hands x_P to the z half through shared memory for T
    constexpr int H = FR_COLS * (1 << B1) / 8;
    __shared__ u64 sm[2][(1 << B1) * FR_COLS];
    __shared__ u64 sx[8][H];
    constexpr u32 log_n = B1 + B2, n2 = 1u << B2;
    const u32 p = blockIdx.x >> (31 - __clz(ngroups)), grp = blockIdx.x & (ngroups - 1);
    const int half = threadIdx.x / H, tl = threadIdx.x % H;
    const int col = tl % FR_COLS, lt = tl / FR_COLS;
    const u32 c = grp * FR_COLS + col;
    const size_t n = (size_t)1 << log_n;
    const u32 prime = half ? a.sp : a.lm1;
    const ModC m = load_mod(tb.mod, prime);
    u64 v[8];
    u64 *zp = a.z + (size_t)p * n;
    const u64 *src = half ? a.acc + ((size_t)p * a.acc_cap + a.acc_cap - 1) * n : zp;
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = src[(size_t)((lt << 3) + i) * n2 + c];
    inv_rounds<B1, 0>(v, ColEx<FR_COLS>{sm[half], col}, lt, 0, 0u, tb.ipsi + ((size_t)prime << log_n), m.q, (int)B2,
                      tb.ipsif + ((size_t)prime << log_n), use_f64(tb, m.q));
    const ulonglong2 ni = __ldg(tb.ninv + prime);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = shoup(v[i], ni.x, ni.y, m.q);
    if (half) {
#pragma unroll
        for (int i = 0; i < 8; ++i) sx[i][tl] = v[i];
    }
    __syncthreads();
    if (half) return;
    const u64 qp = __ldg(&tb.mod[a.sp].q);
    u64 *Tp = a.T + (size_t)p * n;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const u64 zv = v[i], xv = sx[i][tl];
        const size_t e = (size_t)((i << (B1 - 3)) | lt) * n2 + c;  // (x_P < P, z < q_{l-1} < P)
        zp[e] = zv;
        Tp[e] = shoup(xv >= zv ? xv - zv : xv + qp - zv, a.qinv.x, a.qinv.y, qp);
    }
}

template <int B1, int B2>
void fr_tail_impl(const Launch &L, const FrTail &a, u32 np)
{
    const u32 g2 = (1u << B1) / RowGeom<B2>::R, g1 = (1u << B2) / FR_COLS;
    const double nh = (double)np * (1u << (B1 + B2 - 1)), nb = (double)np * (8u << (B1 + B2));
    const double fz = f64_prime(L, a.lm1) ? 1.0 : 0.0, fp = f64_prime(L, a.sp) ? 1.0 : 0.0;
    Work w = nttw(nh * B2, fz, nh * 2, 4 * nb);  // z items: d, acc in; z out
    Work wp = nttw(nh * B2, fp, 0, 2 * nb);
    w.bfly += wp.bfly;
    w.fbfly += wp.fbfly;
    w.bytes += wp.bytes;
    KLAUNCH(L, "fr_rows", w, (k_fr_rows<B2><<<2 * np * g2, 128, 0, L.st>>>(a, *L.tb, g2)));
    Work wc = nttw(nh * B1, fz, nh * 2, 4 * nb);  // z in/out; acc_P in, T out
    Work wcp = nttw(nh * B1, fp, nh * 4, 0);
    wc.bfly += wcp.bfly;
    wc.fbfly += wcp.fbfly;
    KLAUNCH(L, "fr_cols", wc, (k_fr_cols<B1, B2><<<np * g1, 2 * FR_COLS * (1 << B1) / 8, 0, L.st>>>(a, *L.tb, g1)));
}
}  // namespace

void launch_fr_tail(const Launch &L, const u64 *d, u32 d_cap, u64 *acc, u32 acc_cap, u64 *z, u64 *T, u32 np,
                    u32 lm1, u32 sp, ulonglong2 pm, ulonglong2 qinv)
{
    if (!np) return;
    const FrTail a{d, d_cap, acc, acc_cap, z, T, lm1, sp, pm, qinv};
#define CALLFR(b1, b2) fr_tail_impl<b1, b2>(L, a, np)
    CKKS_DISPATCH_LOGN(L.tb->log_n, CALLFR)
#undef CALLFR
}
namespace {
}  // namespace

// ---- compact switching-key rows (launch_key_compact) -------------------------------------------
__global__ void __launch_bounds__(256) k_key_compact(const u64 *tmp, u64 *key, u32 limb, u32 nrows, u32 Lk1,
                                                     u32 log_n, int inverse)
{
    const size_t n = (size_t)1 << log_n, tot = (size_t)nrows << log_n;
    for (size_t x = (size_t)blockIdx.x * blockDim.x + threadIdx.x; x < tot; x += (size_t)gridDim.x * blockDim.x) {
        const size_t row = x >> log_n, k = x & (n - 1);
        u64 *slot = key + (row * Lk1 + limb) * n;
        const u64 *src = tmp + (row << log_n);
        if (!inverse) {
            const u64 v = src[k];
            reinterpret_cast<unsigned *>(slot)[k] = (unsigned)v;
            reinterpret_cast<unsigned char *>(slot)[4 * n + k] = (unsigned char)(v >> 32);
        } else {
            const unsigned char *b = reinterpret_cast<const unsigned char *>(src);
            slot[k] = (u64)reinterpret_cast<const unsigned *>(b)[k] | ((u64)b[4 * n + k] << 32);
        }
    }
}

void launch_key_compact(const Launch &L, u64 *key, const u32 *limbs_host, u32 nl, u32 nrows, u32 Lk1, bool inverse,
                        u64 *tmp)
{
    const size_t n = (size_t)1 << L.tb->log_n;
    const size_t tot = (size_t)nrows * n;
    const u32 blocks = (u32)std::min<size_t>((tot + 255) / 256, (size_t)L.n_sm * 16);
    for (u32 i = 0; i < nl; ++i) {  // gather the limb's rows, then rewrite them in place
        const u32 limb = limbs_host[i];
        cudaMemcpy2DAsync(tmp, n * 8, key + (size_t)limb * n, (size_t)Lk1 * n * 8, n * 8, nrows,
                          cudaMemcpyDeviceToDevice, L.st);
        KLAUNCH(L, "key_compact", (Work{0, 0, 16.0 * (double)tot, 0}),
                (k_key_compact<<<blocks, 256, 0, L.st>>>(tmp, key, limb, nrows, Lk1, L.tb->log_n, inverse ? 1 : 0)));
    }
}
