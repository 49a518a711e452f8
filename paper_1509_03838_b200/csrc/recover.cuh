// recover.cuh -- per-position recovery of all m outputs from m-1 entangled ones.
//
// Restates codec._disentangle_reference / _kernels.disentangle_kernel
// (/root/reference/pkg/src/nent/codec.py:89-107, _kernels.py:33-67):
//
//   pivot  = sum_{t=0}^{m-2} (-1)^t delta_{r+1+t} << (m-2-t) l
//          = (d_r << (m-1) l) + (-1)^m d_{r-1}
//   v      = sign_extend(pivot, (m-1) l);  d_{r-1} = (-1)^m v   (m odd -> -v)
//   d_r    = (pivot - v) >> (m-1) l
//   d_{r+t}= delta_{r+t} - (d_{r+t-1} << l),  t = 1..m-2
//
// narrow (w <= 32): pivot in wrapping int64, exactly like the numba kernel, so
// even inconsistent input (e.g. a skipped kernel self-entanglement) gives the
// reference's bits.  wide (w > 32): pivot exact in 128 bits (the reference's
// Python-int path); d_r not fitting int64 is reported as overflow (the
// reference raises OverflowError when storing it).
//
// Arrays are ROTATED so runtime r never indexes a register array:
//   rot[t]  = delta_{(r+1+t) mod m}, t = 0..m-2     (delta_r is never an input)
//   orot[t] = d_{(r+t) mod m},       t = 0..m-1
#pragma once
#include "common.cuh"

namespace nent {

template <int MT>
__device__ __forceinline__ bool recover_rot(const int64_t* rot, int m, int l, bool wide,
                                            int64_t* orot) {
  const int M = MT > 0 ? MT : m;
  const int low = (M - 1) * l;
  const uint64_t mask = (((uint64_t)1) << low) - 1;  // low <= 63
  const uint64_t sbit = ((uint64_t)1) << (low - 1);
  bool overflow = false;
  int64_t dr, v;
  if (!wide) {
    uint64_t acc = (uint64_t)rot[0] << ((M - 2) * l);
#pragma unroll
    for (int t = 1; t < M - 1; ++t) {
      uint64_t term = (uint64_t)rot[t] << ((M - 2 - t) * l);
      acc = (t & 1) ? acc - term : acc + term;
    }
    v = (int64_t)(((acc & mask) ^ sbit) - sbit);
    dr = (int64_t)(acc - (uint64_t)v) >> low;
  } else {
    // exact while |pivot| < 2^127; unsigned so the shifts are well defined
    typedef unsigned __int128 u128;
    u128 acc = (u128)(__int128)rot[0] << ((M - 2) * l);
#pragma unroll
    for (int t = 1; t < M - 1; ++t) {
      u128 term = (u128)(__int128)rot[t] << ((M - 2 - t) * l);
      acc = (t & 1) ? acc - term : acc + term;
    }
    v = (int64_t)((((uint64_t)acc & mask) ^ sbit) - sbit);
    __int128 q = (__int128)(acc - (u128)(__int128)v) >> low;
    overflow = (q < (__int128)INT64_MIN) || (q > (__int128)INT64_MAX);
    dr = (int64_t)q;
  }
  orot[M - 1] = (M & 1) ? wneg(v) : v;
  orot[0] = dr;
  int64_t prev = dr;
#pragma unroll
  for (int t = 1; t < M - 1; ++t) {
    prev = wsub(rot[t - 1], wshl(prev, l));
    orot[t] = prev;
  }
  return overflow;
}

// Select dl[(base + t) mod MT] for compile-time MT with runtime base, without
// dynamic register indexing.
template <int MT>
__device__ __forceinline__ int64_t select_mod(const int64_t (&dl)[MT], int idx) {
  int64_t v = 0;
#pragma unroll
  for (int s = 0; s < MT; ++s) v = (s == idx) ? dl[s] : v;
  return v;
}

// Full recovery from a per-stream register array dl[s] = delta_s.  pivot r in
// [0, MT); dl[r] is not used.  Writes orot (rotated) and returns overflow.
template <int MT>
__device__ __forceinline__ bool recover_regs(const int64_t (&dl)[MT], int r, int l, bool wide,
                                             int64_t (&orot)[MT]) {
  int64_t rot[MT];
#pragma unroll
  for (int t = 0; t < MT - 1; ++t) {
    int idx = r + 1 + t;
    idx -= (idx >= MT) ? MT : 0;
    idx -= (idx >= MT) ? MT : 0;
    rot[t] = select_mod<MT>(dl, idx);
  }
  rot[MT - 1] = 0;
  return recover_rot<MT>(rot, MT, l, wide, orot);
}

// Recovery for CONSISTENT entangled words (delta_i = (d_{i-1} << l) + d_i with
// every d fitting its word), as the fused kernels produce from admitted
// inputs: the low (m-1)l pivot bits are exact under 64-bit wrap-around for any
// w <= 64, giving d_{r-1}; the rest follow backwards exactly,
//   d_{j-1} = (delta_j - d_j) >> l,   j = r-1, r-2, ..., r+1,
// so no 128-bit pivot is needed even for w = 64.  Results equal the
// reference formula on such input; the fused kernels' redundant-stream check
// flags any input that is not consistent.
template <int MT>
__device__ __forceinline__ void recover_rot_valid(const int64_t* rot, int l, int64_t (&orot)[MT]) {
  const int low = (MT - 1) * l;
  const uint64_t mask = (((uint64_t)1) << low) - 1;
  const uint64_t sbit = ((uint64_t)1) << (low - 1);
  uint64_t acc = (uint64_t)rot[0] << ((MT - 2) * l);
#pragma unroll
  for (int t = 1; t < MT - 1; ++t) {
    const uint64_t term = (uint64_t)rot[t] << ((MT - 2 - t) * l);
    acc = (t & 1) ? acc - term : acc + term;
  }
  const int64_t v = (int64_t)(((acc & mask) ^ sbit) - sbit);
  orot[MT - 1] = (MT & 1) ? wneg(v) : v;
#pragma unroll
  for (int t = MT - 1; t >= 1; --t) orot[t - 1] = wsub(rot[t - 1], orot[t]) >> l;
}

template <int MT>
__device__ __forceinline__ void recover_regs_valid(const int64_t (&dl)[MT], int r, int l,
                                                   int64_t (&orot)[MT]) {
  int64_t rot[MT];
#pragma unroll
  for (int t = 0; t < MT - 1; ++t) {
    int idx = r + 1 + t;
    idx -= (idx >= MT) ? MT : 0;
    idx -= (idx >= MT) ? MT : 0;
    rot[t] = select_mod<MT>(dl, idx);
  }
  recover_rot_valid<MT>(rot, l, orot);
}

}  // namespace nent
