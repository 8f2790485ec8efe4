// Warp-cooperative multi-precision Montgomery arithmetic (one warp per bignum).
//
// A bignum of L = 32*LPL 32-bit limbs lives in one warp: lane l holds limbs
// [l*LPL, l*LPL + LPL) in registers. Moduli N are odd and N < R = 2^(32 L);
// shorter moduli are zero-extended (a 768-bit m^2 runs with LPL = 2).
//
// mont_mul is CIOS (operand scanning): for each limb a_i of a,
//   T += a_i * b;  u = T_0 * n' mod 2^32;  T += u * N;  T >>= 32.
// Per lane the running T is kept in a redundant form: LPL limbs plus a small
// "spill" word s (value at position (l+1)*LPL, owed to the next lane), which
// is folded into the lane's top limb when the window shifts down. Only
// lane 0's t[0] must be exact to form u, and it is: nothing lands below it.
// After the loop the spills are resolved with one ballot-based carry-
// lookahead, and a final conditional subtraction makes the result canonical.
//
// Used by: the Paillier multi-exponentiation (paillier.py:134-193), the
// answer reduction mod m (protocol.py:348-350) and the COMBINED response
// (protocol.py:354-358, paillier.py:104-123).
#pragma once
#include "zpir_common.cuh"

namespace zpir {

template <int LPL>
__device__ __forceinline__ void big_load(uint32_t (&x)[LPL], const uint32_t* __restrict__ p, int lane) {
  const uint32_t* q = p + lane * LPL;
  if constexpr (LPL % 4 == 0) {
#pragma unroll
    for (int i = 0; i < LPL; i += 4) {
      uint4 v = *reinterpret_cast<const uint4*>(q + i);
      x[i] = v.x; x[i + 1] = v.y; x[i + 2] = v.z; x[i + 3] = v.w;
    }
  } else if constexpr (LPL % 2 == 0) {
#pragma unroll
    for (int i = 0; i < LPL; i += 2) {
      uint2 v = *reinterpret_cast<const uint2*>(q + i);
      x[i] = v.x; x[i + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < LPL; ++i) x[i] = q[i];
  }
}

template <int LPL>
__device__ __forceinline__ void big_store(uint32_t* __restrict__ p, const uint32_t (&x)[LPL], int lane) {
  uint32_t* q = p + lane * LPL;
  if constexpr (LPL % 4 == 0) {
#pragma unroll
    for (int i = 0; i < LPL; i += 4)
      *reinterpret_cast<uint4*>(q + i) = make_uint4(x[i], x[i + 1], x[i + 2], x[i + 3]);
  } else if constexpr (LPL % 2 == 0) {
#pragma unroll
    for (int i = 0; i < LPL; i += 2) *reinterpret_cast<uint2*>(q + i) = make_uint2(x[i], x[i + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < LPL; ++i) q[i] = x[i];
  }
}

template <int LPL>
__device__ __forceinline__ void big_set_small(uint32_t (&x)[LPL], uint32_t v, int lane) {
#pragma unroll
  for (int i = 0; i < LPL; ++i) x[i] = 0;
  if (lane == 0) x[0] = v;
}

template <int LPL>
__device__ __forceinline__ void big_copy(uint32_t (&d)[LPL], const uint32_t (&s)[LPL]) {
#pragma unroll
  for (int i = 0; i < LPL; ++i) d[i] = s[i];
}

// Carry into each lane of a warp-wide ripple, from per-lane generate/propagate
// bits: with a = G, b = G|P the carries of the binary sum a + b are exactly
// c_{i+1} = g_i | (p_i & c_i). Returns this lane's carry-in; *out = carry out
// of lane 31.
__device__ __forceinline__ uint32_t lane_carry_in(bool g, bool p, int lane, uint32_t* out) {
  const uint32_t G = __ballot_sync(ZPIR_FULL, g);
  const uint32_t B = G | __ballot_sync(ZPIR_FULL, p);
  const uint64_t s = (uint64_t)G + (uint64_t)B;
  const uint32_t c = (uint32_t)s ^ G ^ B;
  *out = (uint32_t)(s >> 32);
  return (c >> lane) & 1u;
}

// x += cin (0/1) within a lane; returns carry out.
template <int LPL>
__device__ __forceinline__ uint32_t lane_inc(uint32_t (&x)[LPL], uint32_t cin) {
#pragma unroll
  for (int i = 0; i < LPL; ++i) {
    const uint32_t v = x[i] + cin;
    cin = (cin && v == 0) ? 1u : 0u;
    x[i] = v;
  }
  return cin;
}

// x -= bin (0/1) within a lane.
template <int LPL>
__device__ __forceinline__ void lane_dec(uint32_t (&x)[LPL], uint32_t bin) {
#pragma unroll
  for (int i = 0; i < LPL; ++i) {
    const uint32_t v = x[i] - bin;
    bin = (bin && x[i] == 0) ? 1u : 0u;
    x[i] = v;
  }
}

template <int LPL>
__device__ __forceinline__ bool lane_all(const uint32_t (&x)[LPL], uint32_t v) {
  bool r = true;
#pragma unroll
  for (int i = 0; i < LPL; ++i) r = r && (x[i] == v);
  return r;
}

// Warp-wide x = x + y (both L-limb); returns the carry out of the top limb.
template <int LPL>
__device__ __forceinline__ uint32_t big_add(uint32_t (&x)[LPL], const uint32_t (&y)[LPL], int lane) {
  uint64_t c = 0;
#pragma unroll
  for (int i = 0; i < LPL; ++i) {
    c += (uint64_t)x[i] + y[i];
    x[i] = (uint32_t)c;
    c >>= 32;
  }
  const bool g = c != 0;
  const bool p = lane_all(x, 0xffffffffu);
  uint32_t out;
  const uint32_t cin = lane_carry_in(g, p, lane, &out);
  lane_inc(x, cin);
  return out;
}

// Canonicalise V = x + top * R (V < 2N) to V mod N, in place.
template <int LPL>
__device__ __forceinline__ void big_cond_sub(uint32_t (&x)[LPL], uint32_t top,
                                             const uint32_t (&n)[LPL], int lane) {
  uint32_t d[LPL];
  uint32_t br = 0;
#pragma unroll
  for (int i = 0; i < LPL; ++i) {
    const uint64_t v = (uint64_t)x[i] - n[i] - br;
    d[i] = (uint32_t)v;
    br = (uint32_t)(v >> 63);
  }
  const bool g = br != 0;
  const bool p = lane_all(d, 0u) && !g;
  uint32_t bout;
  const uint32_t bin = lane_carry_in(g, p, lane, &bout);
  lane_dec(d, bin);
  const bool ge = top >= bout;  // V - N = d + (top - bout) * R
#pragma unroll
  for (int i = 0; i < LPL; ++i) x[i] = ge ? d[i] : x[i];
}

// V = x + h * R (h small) to V mod N in place, given a quotient estimate q with
// q <= floor(V / N) <= q + 1 (callers divide the top bits of V by the top bits
// of N plus one): V - q N < 2N, then one conditional subtraction.
template <int LPL>
__device__ __forceinline__ void big_reduce_top(uint32_t (&x)[LPL], uint32_t h, uint32_t q,
                                               const uint32_t (&n)[LPL], int lane) {
  // M = q * N: lane-local limbs, the lane's high word owed to the next lane
  uint32_t m[LPL];
  uint64_t c = 0;
#pragma unroll
  for (int k = 0; k < LPL; ++k) {
    c += (uint64_t)q * n[k];
    m[k] = (uint32_t)c;
    c >>= 32;
  }
  const uint32_t hi = (uint32_t)c;
  uint32_t lo = __shfl_up_sync(ZPIR_FULL, hi, 1);
  lo = lane == 0 ? 0u : lo;
  c = lo;
#pragma unroll
  for (int k = 0; k < LPL; ++k) {
    c += m[k];
    m[k] = (uint32_t)c;
    c >>= 32;
  }
  uint32_t cout;
  const uint32_t cin = lane_carry_in(c != 0, lane_all(m, 0xffffffffu), lane, &cout);
  lane_inc(m, cin);
  const uint32_t mtop = __shfl_sync(ZPIR_FULL, hi, 31) + cout;   // limb L of M
  // x <- x - M, borrow out of the top limb into h
  uint32_t br = 0;
#pragma unroll
  for (int k = 0; k < LPL; ++k) {
    const uint64_t v = (uint64_t)x[k] - m[k] - br;
    x[k] = (uint32_t)v;
    br = (uint32_t)(v >> 63);
  }
  const bool g = br != 0;
  uint32_t bout;
  const uint32_t bin = lane_carry_in(g, lane_all(x, 0u) && !g, lane, &bout);
  lane_dec(x, bin);
  big_cond_sub(x, h - mtop - bout, n, lane);
}

// t += x * y with 64-bit products (compiles to IMAD.WIDE.U32 chains); measured
// fewer SASS instructions than an explicit PTX carry chain (measured round 1).
template <int LPL>
__device__ __forceinline__ void mac_row_c(uint32_t (&t)[LPL], uint32_t& s0, uint32_t& s1,
                                          uint32_t x, const uint32_t (&y)[LPL]) {
  uint64_t c = 0;
#pragma unroll
  for (int k = 0; k < LPL; ++k) {
    const uint64_t p = (uint64_t)x * y[k] + t[k] + c;  // <= 2^64 - 1
    t[k] = (uint32_t)p;
    c = p >> 32;
  }
  const uint64_t s = (((uint64_t)s1 << 32) | s0) + c;
  s0 = (uint32_t)s;
  s1 = (uint32_t)(s >> 32);
}

// t += x * y (lane-local LPL limbs); the carry out of the lane goes to the
// 64-bit spill (s1:s0).
template <int LPL>
__device__ __forceinline__ void mac_row(uint32_t (&t)[LPL], uint32_t& s0, uint32_t& s1,
                                        uint32_t x, const uint32_t (&y)[LPL]) {
  mac_row_c<LPL>(t, s0, s1, x, y);    // IMAD.WIDE.U32 + 64-bit adds: fewest instructions
}

// r = a * b * R^-1 mod N, canonical. Requires a < R, b < N (then T < 2N).
// r may alias a or b. UNR unrolls the limb-broadcast loop: 1 for the
// IMAD-throughput-bound kernels; 4 for latency-bound callers with few warps per
// SM (slot_combine's 2016-deep Horner chain per group), so the independent
// a-limb broadcasts of later steps overlap the u-chain.
template <int LPL, int UNR = 1>
__device__ __forceinline__ void mont_mul(uint32_t (&r)[LPL], const uint32_t (&a)[LPL],
                                         const uint32_t (&b)[LPL], const uint32_t (&n)[LPL],
                                         uint32_t np, int lane) {
  uint32_t t[LPL];
#pragma unroll
  for (int i = 0; i < LPL; ++i) t[i] = 0;
  uint32_t s0 = 0, s1 = 0;
#pragma unroll UNR
  for (int src = 0; src < 32; ++src) {
#pragma unroll
    for (int rr = 0; rr < LPL; ++rr) {
      const uint32_t ai = __shfl_sync(ZPIR_FULL, a[rr], src);
      mac_row(t, s0, s1, ai, b);
      const uint32_t u = __shfl_sync(ZPIR_FULL, t[0] * np, 0);
      mac_row(t, s0, s1, u, n);
      uint32_t nx = __shfl_down_sync(ZPIR_FULL, t[0], 1);
      nx = (lane == 31) ? 0u : nx;
#pragma unroll
      for (int k = 0; k < LPL - 1; ++k) t[k] = t[k + 1];
      const uint64_t z = (uint64_t)nx + s0;
      t[LPL - 1] = (uint32_t)z;
      s0 = s1 + (uint32_t)(z >> 32);
      s1 = 0;
    }
  }
  // resolve the pending spills: lane l owes s0 to lane l+1's lowest limb
  uint32_t sp = __shfl_up_sync(ZPIR_FULL, s0, 1);
  sp = (lane == 0) ? 0u : sp;
  uint64_t c = sp;
#pragma unroll
  for (int i = 0; i < LPL; ++i) {
    c += t[i];
    t[i] = (uint32_t)c;
    c >>= 32;
  }
  const bool g = c != 0;
  const bool p = lane_all(t, 0xffffffffu);
  uint32_t cout;
  const uint32_t cin = lane_carry_in(g, p, lane, &cout);
  lane_inc(t, cin);
  const uint32_t top = __shfl_sync(ZPIR_FULL, s0, 31) + cout;
  big_cond_sub(t, top, n, lane);
#pragma unroll
  for (int i = 0; i < LPL; ++i) r[i] = t[i];
}

}  // namespace zpir
