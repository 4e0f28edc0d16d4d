// hostmath.h -- host-side number theory and CKKS encode/decode for libckks.
// Independent of oracle/ (no shared code): prime scan, roots, Shoup companions,
// the special FFT of the canonical embedding, and multi-precision CRT for decode.
#pragma once
#include <complex>
#include <cstdint>
#include <string>
#include <vector>

namespace hm {
typedef uint64_t u64;
typedef unsigned __int128 u128;

u64 mulmod(u64 a, u64 b, u64 q);
u64 powmod(u64 b, u64 e, u64 q);
u64 invmod(u64 a, u64 q);            // q prime
bool is_prime(u64 n);                // deterministic Miller-Rabin (bases 2..37)
u64 shoup(u64 w, u64 q);             // floor(w 2^64 / q)
// Chain rule of ckks_params (include/ckks.h): P first from its bit scan, then q_i in order.
bool prime_chain(uint32_t log_n, uint32_t L, const uint32_t *limb_bits, uint32_t special_bits, uint32_t K,
                 std::vector<u64> &out /* q_0..q_{L-1}, p_0..p_{K-1} */, std::string &err);
u64 primitive_2n_root(u64 q, uint32_t log_n);  // some psi with psi^N = -1
uint32_t bitrev(uint32_t x, uint32_t bits);

// Canonical embedding (reading A12): slot j <-> zeta^{5^j}, zeta = e^{i pi/N}.
// encode: coefficients m_k = round(Re(...)) of the real polynomial interpolating Delta z.
void encode(const std::complex<double> *z, size_t nslots, double scale, uint32_t log_n, std::vector<double> &coef);
// decode: slots from real (centred) coefficients divided by scale.
void decode(const std::vector<double> &coef, double scale, uint32_t log_n, std::vector<std::complex<double>> &z);
// centred CRT value of residues (one coefficient) as a double, given precomputed data
struct Crt {
    std::vector<u64> q;
    std::vector<std::vector<u64>> Qi;  // Q / q_i as little-endian words
    std::vector<u64> Qi_inv;           // (Q / q_i)^{-1} mod q_i
    std::vector<u64> Q, Qhalf;
    void init(const std::vector<u64> &primes);
    double centred(const u64 *res, size_t stride) const;  // res[i * stride] = residue mod q_i
};
}  // namespace hm
