// rng.cuh -- counter-based random keys of the WRS node selection (device side).
//
// Written from the contract in DESIGN.md (R13, R14), independently of the oracle.
// Paper: Sec. 4.2.2 -- one uniform r in (0,1) per
// considered node, key k = (1/w) log2 r, where the paper keeps a per-thread
// generator state and uses the MUFU __log2f.  Here the generator is stateless
// (Philox4x32-10, so any thread can draw any (node, step, ant, iteration)
// number without carrying state) and the logarithm is a fixed fp32 polynomial
// evaluated with explicit round-to-nearest intrinsics, so the result is
// reproducible bit for bit on the CPU.
#pragma once
#include <cstdint>

namespace mmas {

struct PhiloxKey {
    uint32_t k0, k1;
};

// Philox4x32-10 (Salmon et al., SC'11): 10 rounds of two 32x32->64 multiplies,
// key bumped by the Weyl constants between rounds.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, PhiloxKey key) {
    uint32_t k0 = key.k0, k1 = key.k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint32_t lo0 = 0xD2511F53u * c.x;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    }
    return c;
}

// u = (2*(x>>9)+1) * 2^-24: 23 random bits, exactly representable, in the open
// interval (0,1) that A-Res and the log key need.
// Built without an int->float conversion (those issue on the narrow XU pipe, which
// the construction kernels would otherwise saturate): 1 + j 2^-23 from the mantissa
// bits, minus (1 - 2^-24); the difference (2j+1) 2^-24 has <= 24 significant bits,
// so the subtraction is exact and the value equals (float)(2j+1) * 2^-24 bit for bit.
__device__ __forceinline__ float uniform_open(uint32_t x) {
    return __fsub_rn(__uint_as_float(0x3F800000u | (x >> 9)), 0.99999994039535522461f);
}

// 1 - u for the same x, exactly (1 - u = (2^24 - 2j - 1) 2^-24 has 24 significant bits):
// 1 + (2^23 - 1 - j) 2^-23 = 2 - (j+1) 2^-23 from the bits 0x3FFFFFFF - j, minus (1 - 2^-24).
// (The pruned scans need 1 - u for every city and u itself only for the few survivors.)
__device__ __forceinline__ float one_minus_uniform_open(uint32_t x) {
    return __fsub_rn(__uint_as_float(0x3FFFFFFFu - (x >> 9)), 0.99999994039535522461f);
}

// det_log2 (R14): u = 2^e * m, m in [sqrt(1/2), sqrt(2)), f = m - 1 (exact),
// log2 u = e + f * P(f), P of degree 8 (coefficients frozen in DESIGN.md).
// Valid for normal u > 0, which covers every value uniform_open() produces.
__device__ __forceinline__ float det_log2(float u) {
    const uint32_t b = __float_as_uint(u);
    const uint32_t mant = b & 0x007FFFFFu;
    int e = (int)(b >> 23) - 127;
    uint32_t mb = mant | 0x3F800000u;                        // m in [1, 2)
    if (mant > 0x003504F3u) {                                // m > (float)sqrt(2): use m/2
        mb = mant | 0x3F000000u;
        e += 1;
    }
    const float f = __fsub_rn(__uint_as_float(mb), 1.0f);
    float p = 0.12583690881729126f;
    p = __fmaf_rn(p, f, -0.20726971328258514f);
    p = __fmaf_rn(p, f, 0.21571563184261322f);
    p = __fmaf_rn(p, f, -0.23894482851028442f);
    p = __fmaf_rn(p, f, 0.28791624307632446f);
    p = __fmaf_rn(p, f, -0.3607036769390106f);
    p = __fmaf_rn(p, f, 0.48091062903404236f);
    p = __fmaf_rn(p, f, -0.7213473320007324f);
    p = __fmaf_rn(p, f, 1.4426950216293335f);
    // (float)e without I2F: 1.5 * 2^23 + e is exact in the significand for |e| < 2^22
    const float ef = __fsub_rn(__int_as_float(0x4B400000 + e), 12582912.0f);
    return __fmaf_rn(f, p, ef);
}

// det_log2 in two parts (the same operations in the same order, so bit-identical): the
// construction kernels place the halves in different latency windows of a step.
struct Log2Part {
    float f, p, ef;
};
__device__ __forceinline__ Log2Part det_log2_a(float u) {
    const uint32_t b = __float_as_uint(u);
    const uint32_t mant = b & 0x007FFFFFu;
    int e = (int)(b >> 23) - 127;
    uint32_t mb = mant | 0x3F800000u;
    if (mant > 0x003504F3u) {
        mb = mant | 0x3F000000u;
        e += 1;
    }
    Log2Part r;
    r.f = __fsub_rn(__uint_as_float(mb), 1.0f);
    float p = 0.12583690881729126f;
    p = __fmaf_rn(p, r.f, -0.20726971328258514f);
    p = __fmaf_rn(p, r.f, 0.21571563184261322f);
    p = __fmaf_rn(p, r.f, -0.23894482851028442f);
    p = __fmaf_rn(p, r.f, 0.28791624307632446f);
    r.p = p;
    r.ef = __fsub_rn(__int_as_float(0x4B400000 + e), 12582912.0f);
    return r;
}
__device__ __forceinline__ float det_log2_b(const Log2Part& r) {
    float p = r.p;
    p = __fmaf_rn(p, r.f, -0.3607036769390106f);
    p = __fmaf_rn(p, r.f, 0.48091062903404236f);
    p = __fmaf_rn(p, r.f, -0.7213473320007324f);
    p = __fmaf_rn(p, r.f, 1.4426950216293335f);
    return __fmaf_rn(r.f, p, r.ef);
}

// Counter layouts (R13).  x2 = global ant id, x3 = global iteration.
__device__ __forceinline__ uint4 ctr_start(uint32_t ant, uint32_t iter) {
    return make_uint4(0x80000000u, 0u, ant, iter);
}
// candidate slot k, step group s>>2 -> word (s & 3) is slot k's uniform at step s
__device__ __forceinline__ uint4 ctr_slot(uint32_t slot, uint32_t step_group, uint32_t ant, uint32_t iter) {
    return make_uint4(slot, step_group, ant, iter);
}
// city group c>>2 at step s -> word (c & 3) is city c's uniform
__device__ __forceinline__ uint4 ctr_city(uint32_t city_group, uint32_t step, uint32_t ant, uint32_t iter) {
    return make_uint4(0x40000000u | city_group, step, ant, iter);
}

}  // namespace mmas
