// hostmath.cpp -- see hostmath.h.
#include "hostmath.h"

#include <algorithm>
#include <cmath>

namespace hm {

u64 mulmod(u64 a, u64 b, u64 q) { return (u64)((u128)a * b % q); }

u64 powmod(u64 b, u64 e, u64 q)
{
    u64 r = 1 % q;
    b %= q;
    for (; e; e >>= 1) {
        if (e & 1) r = mulmod(r, b, q);
        b = mulmod(b, b, q);
    }
    return r;
}

u64 invmod(u64 a, u64 q) { return powmod(a % q, q - 2, q); }

bool is_prime(u64 n)
{
    const u64 small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return false;
    for (u64 p : small) {
        if (n % p == 0) return n == p;
    }
    u64 d = n - 1;
    int s = 0;
    while (!(d & 1)) {
        d >>= 1;
        ++s;
    }
    for (u64 a : small) {
        u64 x = powmod(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int r = 1; r < s && comp; ++r) {
            x = mulmod(x, x, n);
            if (x == n - 1) comp = false;
        }
        if (comp) return false;
    }
    return true;
}

u64 shoup(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }

bool prime_chain(uint32_t log_n, uint32_t L, const uint32_t *limb_bits, uint32_t special_bits, uint32_t K,
                 std::vector<u64> &out, std::string &err)
{
    const u64 step = (u64)2 << log_n;
    std::vector<std::pair<uint32_t, u64>> cursor;  // bits -> next candidate
    auto next = [&](uint32_t bits, u64 &p) -> bool {
        if (bits < 2 || bits > 62) {
            err = "prime bit size must be in [2, 62]";
            return false;
        }
        auto it = std::find_if(cursor.begin(), cursor.end(), [&](auto &c) { return c.first == bits; });
        if (it == cursor.end()) {
            u64 top = ((u64)1 << bits) - 1;
            cursor.push_back({bits, (top - 1) / step * step + 1});
            it = cursor.end() - 1;
        }
        for (u64 x = it->second;; x -= step) {
            if (x <= step) {
                err = "prime exhaustion";
                return false;
            }
            if (is_prime(x)) {
                p = x;
                it->second = x - step;
                return true;
            }
        }
    };
    out.assign(L + K, 0);
    u64 p;
    for (uint32_t k = 0; k < K; ++k) {
        if (!next(special_bits, p)) return false;
        out[L + k] = p;
    }
    for (uint32_t i = 0; i < L; ++i) {
        if (!next(limb_bits[i], p)) return false;
        out[i] = p;
    }
    return true;
}

u64 primitive_2n_root(u64 q, uint32_t log_n)
{
    const u64 n = (u64)1 << log_n;
    if ((q - 1) % (2 * n)) return 0;
    for (u64 x = 2; x < q; ++x) {
        u64 g = powmod(x, (q - 1) / (2 * n), q);
        if (powmod(g, n, q) == q - 1) return g;
    }
    return 0;
}

uint32_t bitrev(uint32_t x, uint32_t bits)
{
    uint32_t r = 0;
    for (uint32_t i = 0; i < bits; ++i) r |= ((x >> i) & 1u) << (bits - 1 - i);
    return r;
}

// in-place iterative radix-2 complex FFT, sign = -1: X_s = sum x_k e^{-2 pi i s k / n}
static void fft(std::vector<std::complex<double>> &a, int sign)
{
    const size_t n = a.size();
    for (size_t i = 1, j = 0; i < n; ++i) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(a[i], a[j]);
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        const size_t h = len / 2;
        std::vector<std::complex<double>> w(h);
        for (size_t k = 0; k < h; ++k) {
            const double ang = sign * 2.0 * M_PI * (double)k / (double)len;
            w[k] = std::complex<double>(std::cos(ang), std::sin(ang));
        }
        for (size_t i = 0; i < n; i += len)
            for (size_t k = 0; k < h; ++k) {
                std::complex<double> u = a[i + k], v = a[i + k + h] * w[k];
                a[i + k] = u + v;
                a[i + k + h] = u - v;
            }
    }
}

// m(zeta^{2s+1}) = sum_k (m_k zeta^k) omega^{s k}, omega = e^{2 pi i / N}
void encode(const std::complex<double> *z, size_t nslots, double scale, uint32_t log_n, std::vector<double> &coef)
{
    const size_t n = (size_t)1 << log_n, t = n / 2;
    std::vector<std::complex<double>> B(n, 0.0);
    u64 r = 1;
    for (size_t j = 0; j < t; ++j) {
        std::complex<double> v = j < nslots ? z[j] * scale : 0.0;
        B[(r - 1) / 2] = v;
        B[(2 * n - r - 1) / 2] = std::conj(v);
        r = (r * 5) % (2 * n);
    }
    fft(B, -1);  // b_k N = sum_s B_s omega^{-s k}
    coef.resize(n);
    for (size_t k = 0; k < n; ++k) {
        const double ang = -M_PI * (double)k / (double)n;
        coef[k] = (B[k] * std::complex<double>(std::cos(ang), std::sin(ang))).real() / (double)n;
    }
}

void decode(const std::vector<double> &coef, double scale, uint32_t log_n, std::vector<std::complex<double>> &z)
{
    const size_t n = (size_t)1 << log_n, t = n / 2;
    std::vector<std::complex<double>> b(n);
    for (size_t k = 0; k < n; ++k) {
        const double ang = M_PI * (double)k / (double)n;
        b[k] = coef[k] * std::complex<double>(std::cos(ang), std::sin(ang));
    }
    fft(b, +1);
    z.resize(t);
    u64 r = 1;
    for (size_t j = 0; j < t; ++j) {
        z[j] = b[(r - 1) / 2] / scale;
        r = (r * 5) % (2 * n);
    }
}

// ---- small multi-precision helpers (little-endian u64 words) ----------------------------
static void mp_mul_small(const std::vector<u64> &a, u64 m, std::vector<u64> &out)
{
    out.assign(a.size() + 1, 0);
    u64 carry = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        u128 p = (u128)a[i] * m + carry;
        out[i] = (u64)p;
        carry = (u64)(p >> 64);
    }
    out[a.size()] = carry;
}
static void mp_add(std::vector<u64> &acc, const std::vector<u64> &b)
{
    if (acc.size() < b.size()) acc.resize(b.size(), 0);
    u64 carry = 0;
    for (size_t i = 0; i < acc.size(); ++i) {
        u128 s = (u128)acc[i] + (i < b.size() ? b[i] : 0) + carry;
        acc[i] = (u64)s;
        carry = (u64)(s >> 64);
    }
    if (carry) acc.push_back(carry);
}
static int mp_cmp(const std::vector<u64> &a, const std::vector<u64> &b)
{
    size_t n = std::max(a.size(), b.size());
    for (size_t i = n; i-- > 0;) {
        u64 x = i < a.size() ? a[i] : 0, y = i < b.size() ? b[i] : 0;
        if (x != y) return x < y ? -1 : 1;
    }
    return 0;
}
static void mp_sub(std::vector<u64> &a, const std::vector<u64> &b)  // a -= b, a >= b
{
    u64 borrow = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        u64 y = (i < b.size() ? b[i] : 0);
        u128 d = (u128)a[i] - y - borrow;
        a[i] = (u64)d;
        borrow = (d >> 127) ? 1 : 0;
    }
}
static double mp_to_double(const std::vector<u64> &a)
{
    long double r = 0;
    for (size_t i = a.size(); i-- > 0;) r = r * 18446744073709551616.0L + (long double)a[i];
    return (double)r;
}

void Crt::init(const std::vector<u64> &primes)
{
    q = primes;
    Q = {1};
    for (u64 p : q) {
        std::vector<u64> t;
        mp_mul_small(Q, p, t);
        while (t.size() > 1 && t.back() == 0) t.pop_back();
        Q = t;
    }
    Qi.assign(q.size(), {});
    Qi_inv.assign(q.size(), 0);
    for (size_t i = 0; i < q.size(); ++i) {
        std::vector<u64> acc = {1};
        u64 rmod = 1;
        for (size_t j = 0; j < q.size(); ++j)
            if (j != i) {
                std::vector<u64> t;
                mp_mul_small(acc, q[j], t);
                acc = t;
                rmod = mulmod(rmod, q[j] % q[i], q[i]);
            }
        while (acc.size() > 1 && acc.back() == 0) acc.pop_back();
        Qi[i] = acc;
        Qi_inv[i] = invmod(rmod, q[i]);
    }
    // Qhalf = floor(Q / 2)
    Qhalf = Q;
    u64 carry = 0;
    for (size_t i = Qhalf.size(); i-- > 0;) {
        u64 w = Qhalf[i];
        Qhalf[i] = (w >> 1) | (carry << 63);
        carry = w & 1;
    }
}

double Crt::centred(const u64 *res, size_t stride) const
{
    if (q.size() == 1) {
        u64 x = res[0];
        return x > q[0] / 2 ? -(double)(q[0] - x) : (double)x;
    }
    std::vector<u64> acc = {0}, t;
    for (size_t i = 0; i < q.size(); ++i) {
        u64 y = mulmod(res[i * stride], Qi_inv[i], q[i]);
        mp_mul_small(Qi[i], y, t);
        mp_add(acc, t);
    }
    while (mp_cmp(acc, Q) >= 0) mp_sub(acc, Q);
    if (mp_cmp(acc, Qhalf) > 0) {
        std::vector<u64> neg = Q;
        mp_sub(neg, acc);
        return -mp_to_double(neg);
    }
    return mp_to_double(acc);
}

}  // namespace hm
