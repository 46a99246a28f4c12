// sm_100a kernels of libtoast.
//
// K1 toast_eval_kernel   — one warp per candidate; lane i of the warp owns
//   op (base + i) of a 32-op window that slides over the program in order
//   (H1 decode, H2 materialise, H3 FLOPs, H4 collectives, H5 liveness as a
//   warp inclusive scan + max, H6 score, H7 key).  No tensor cores: there is
//   no dense contraction on this path (SURVEY §8(d) "Roofline").
// K2 toast_rollout_kernel — one warp per rollout: Philox4x32-10 draws, the
//   legal-action bitset distributed one 32-bit word per lane (ballot/popc
//   selection), then the K1 device path on the finished sequence (H8).
//
// Every quantity is an integer until the fixed double epilogue, which uses
// explicit _rn intrinsics (never contracted into FMA) so the score is
// bit-identical to the CPU oracle's.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <string>

#include "toast_internal.h"

namespace toast {

namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// exact division by the product of the axis sizes in subset S (the divisor
// always divides x exactly on this path): (x >> twos) * odd^-1 mod 2^64
__device__ __forceinline__ uint64_t exdiv(const DeviceTables& T, uint64_t x, uint32_t S) {
  return (x >> T.shift[S]) * T.inv[S];
}

__device__ __forceinline__ uint64_t warp_or64(uint64_t v) {
  uint32_t lo = __reduce_or_sync(FULL, (uint32_t)v);
  uint32_t hi = __reduce_or_sync(FULL, (uint32_t)(v >> 32));
  return ((uint64_t)hi << 32) | lo;
}

struct Mat {
  uint32_t masks;   // 4 bits per role
  uint32_t opmask;  // OR of all masks
};

struct OpRec {
  uint32_t loop_begin, res_roles, use_begin, death_begin;
  uint32_t n_loops, rank, rmask, flags, n_death, n_uses;
  uint64_t gbytes;
};

__device__ __forceinline__ OpRec load_op(const DeviceTables& T, uint32_t t) {
  const uint4* p = reinterpret_cast<const uint4*>(T.ops + t);
  uint4 a = __ldg(p), b = __ldg(p + 1);
  OpRec r;
  r.loop_begin = a.x;
  r.n_loops = a.y & 0xFF;
  r.rank = (a.y >> 8) & 0xFF;
  r.rmask = (a.y >> 16) & 0xFF;
  r.flags = a.y >> 24;
  r.res_roles = a.z;
  r.use_begin = a.w;
  r.death_begin = b.x;
  r.n_death = b.y & 0xFFFF;
  r.n_uses = (b.y >> 16) & 0xFF;
  r.gbytes = ((uint64_t)b.w << 32) | b.z;
  return r;
}

// H2 (C9): per-op materialisation.  Events (action position j, role) are
// merged in action order, roles in role order; an axis shards at most one
// loop of the op; divisibility via the loop's div_ok subset mask.
__device__ __forceinline__ Mat materialize(const DeviceTables& T, const uint32_t* __restrict__ acol, uint32_t lb,
                                           uint32_t nl, uint64_t fixed0, uint64_t ones) {
  uint32_t list[MAX_LOOPS_PER_OP], div[MAX_LOOPS_PER_OP];
  uint32_t any = 0;
#pragma unroll
  for (int r = 0; r < MAX_LOOPS_PER_OP; ++r) {
    list[r] = 0;
    div[r] = 0;
    if (r < (int)nl) {
      uint64_t L = __ldg(T.loops + lb + r);
      uint32_t ac = (uint32_t)L & 0x3FF;
      div[r] = (uint32_t)(L >> 12) & 0xFFFF;
      if (ac != NO_ACOLOR) {
        uint32_t li = acol[ac];
        uint32_t did = (uint32_t)(L >> 28) & 0xFFFF;
        if (li && did) {
          uint64_t n0 = __ldg(T.desel + 2 * did), n1 = __ldg(T.desel + 2 * did + 1);
          if ((fixed0 & n0) | (ones & n1)) li = 0;
        }
        list[r] = li;
        any |= li;
      }
    }
  }
  Mat m{0, 0};
  if (!any) return m;
  while (true) {
    int best = -1;
    uint32_t bj = 64;
#pragma unroll
    for (int r = 0; r < MAX_LOOPS_PER_OP; ++r) {
      uint32_t e = list[r];
      if ((e & 0x80) && (e & 31) < bj) { bj = e & 31; best = r; }
    }
    if (best < 0) break;
    uint32_t e = 0, dv = 0;
#pragma unroll
    for (int r = 0; r < MAX_LOOPS_PER_OP; ++r)
      if (r == best) { e = list[r]; dv = div[r]; list[r] = e >> 8; }
    uint32_t A = (e >> 5) & 3;
    uint32_t cur = (m.masks >> (4 * best)) & 15;
    if (!((m.opmask >> A) & 1) && ((dv >> (cur | (1u << A))) & 1)) {
      m.masks |= (1u << A) << (4 * best);
      m.opmask |= 1u << A;
    }
  }
  return m;
}

// per-dim masks (4 bits each) of a site given its role map
__device__ __forceinline__ uint32_t site_masks(uint32_t masks, uint32_t roles, uint32_t rank) {
  uint32_t out = 0;
#pragma unroll
  for (int i = 0; i < MAX_RANK; ++i)
    if (i < (int)rank) out |= ((masks >> (4 * ((roles >> (4 * i)) & 15))) & 15) << (4 * i);
  return out;
}
__device__ __forceinline__ uint32_t dims_or(uint32_t dm) {
  dm |= dm >> 16;
  dm |= dm >> 8;
  dm |= dm >> 4;
  return dm & 15;
}
__device__ __forceinline__ uint32_t roles_or(uint32_t masks, uint32_t rmask) {
  uint32_t out = 0;
#pragma unroll
  for (int r = 0; r < MAX_LOOPS_PER_OP; ++r)
    if ((rmask >> r) & 1) out |= (masks >> (4 * r)) & 15;
  return out;
}
// dim holding axis A in a packed site (-1 if none)
__device__ __forceinline__ int dim_of(uint32_t dm, uint32_t A) {
  uint32_t sel = dm & (0x11111111u << A);
  return sel ? (__ffs(sel) - 1) >> 2 : -1;
}

struct Acc {   // per-warp shared accumulators
  unsigned long long payload[16];
  unsigned int count[16];
};

// one candidate per warp; `sid` = this lane's action id (seq[lane])
__device__ void eval_warp(const DeviceTables& T, uint32_t sid, uint32_t* __restrict__ acol, Acc* __restrict__ acc,
                          unsigned long long* __restrict__ rec, toast_cost* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  // ---------------- H1 decode (C9)
  unsigned zb = __ballot_sync(FULL, sid == 0);
  int stop = zb ? __ffs(zb) - 1 : 32;
  bool active = lane < stop;
  uint32_t status = 0;
  if (__ballot_sync(FULL, lane > stop && sid != 0)) status |= TOAST_ST_NONZERO_AFTER_STOP;
  bool bad = active && (int)sid >= T.n_actions;
  if (__ballot_sync(FULL, bad)) status |= TOAST_ST_BAD_ACTION_ID;
  bool ok = active && !bad;
  uint32_t aw = ok ? __ldg(T.actions + sid) : 0u;
  uint32_t ac = aw & 0x3FF, rr = (aw >> 10) & 0xFF, ax = (aw >> 18) & 3;
  unsigned same = __match_any_sync(FULL, ok ? ((ac << 2) | ax) : (0x80000000u | (uint32_t)lane));
  if (__ballot_sync(FULL, ok && __popc(same) > 1)) status |= TOAST_ST_DUP_COLOR_AXIS;
  uint64_t fx = 0, on = 0;
  if (ok) {
    uint64_t gw = __ldg(T.acol_groups + ac);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      uint32_t gid = (uint32_t)(gw >> (8 * t)) & 0xFF;
      if (gid != 0xFF) {
        fx |= 1ULL << gid;
        if ((rr >> t) & 1) on |= 1ULL << gid;
      }
    }
  }
  uint64_t zr = warp_or64(fx & ~on);
  on = warp_or64(on);
  if (on & zr) status |= TOAST_ST_RES_MISMATCH;
  if (status) {
    if (lane == 0) {
      memset(rec, 0, 256);
      reinterpret_cast<uint32_t*>(rec)[10] = status;
    }
    __syncwarp();
    reinterpret_cast<unsigned long long*>(out)[lane] = rec[lane];
    __syncwarp();
    return;
  }
  unsigned samec = __match_any_sync(FULL, ok ? ac : (0x80000000u | (uint32_t)lane));
  int rank_in_color = __popc(samec & ((1u << lane) - 1u));
  if (ok) atomicOr(acol + ac, (0x80u | (ax << 5) | (uint32_t)lane) << (8 * rank_in_color));
  if (lane < 16) { acc->payload[lane] = 0ULL; acc->count[lane] = 0u; }
  __syncwarp();

  // ---------------- sweep over ops, 32 at a time
  uint64_t key = 0, flo = 0, fhi = 0;
  long long carry = 0, peak = 0;
  for (int base = 0; base < T.n_ops; base += 32) {
    const int t = base + lane;
    long long delta = 0, inop = 0;
    const bool live = t < T.n_ops;
    if (live) {
      OpRec op = load_op(T, (uint32_t)t);
      Mat me = materialize(T, acol, op.loop_begin, op.n_loops, zr, on);
      // H7 key (C14)
      if (me.masks) {
#pragma unroll
        for (int r = 0; r < MAX_LOOPS_PER_OP; ++r) {
          uint32_t mk = (me.masks >> (4 * r)) & 15;
          if (mk) key += mix64(((uint64_t)(op.loop_begin + r) << 8) | mk);
        }
      }
      // H3 FLOPs (C10)
      if (op.flags & 1) {
        uint64_t f = exdiv(T, __ldg(T.gflops + t), me.opmask);
        flo += f;
        fhi += (flo < f) ? 1 : 0;
      }
      long long res = 0;
      if (!(op.flags & 2)) res = (long long)exdiv(T, op.gbytes, dims_or(site_masks(me.masks, op.res_roles, op.rank)));
      // H4 collectives per use edge (C11)
      uint32_t Uk[MAX_USES_PER_OP], vk[MAX_USES_PER_OP];
      long long gk[MAX_USES_PER_OP];
      long long temp_total = 0;
#pragma unroll
      for (int k = 0; k < MAX_USES_PER_OP; ++k) {
        Uk[k] = 0; vk[k] = 0xFFFFFFFFu; gk[k] = 0;
        if (k < (int)op.n_uses) {
          uint2 uw = __ldg(reinterpret_cast<const uint2*>(T.uses + op.use_begin + k));
          uint32_t v = uw.x;
          OpRec dop = load_op(T, v);
          uint32_t U = site_masks(me.masks, uw.y, dop.rank);
          Uk[k] = U;
          vk[k] = v;
          bool dup = false;
#pragma unroll
          for (int k2 = 0; k2 < k; ++k2) dup |= (vk[k2] == v && Uk[k2] == U);
          if (!dup) {
            Mat dm = materialize(T, acol, dop.loop_begin, dop.n_loops, zr, on);
            uint32_t D = site_masks(dm.masks, dop.res_roles, dop.rank);
            uint32_t P = roles_or(dm.masks, dop.rmask);
            if (D != U || P != 0) {
              uint32_t Dp = dims_or(D), Up = dims_or(U);
              uint64_t size = exdiv(T, dop.gbytes, Dp);
              for (int A = 0; A < T.n_axes; ++A) {          // phase 1: AG / A2A
                int dD = dim_of(D, A);
                if (dD < 0) continue;
                int dU = dim_of(U, A);
                if (dD == dU) continue;
                if (dU >= 0) {
                  atomicAdd(&acc->payload[A * 4 + TOAST_A2A], (unsigned long long)size);
                  atomicAdd(&acc->count[A * 4 + TOAST_A2A], 1u);
                } else {
                  atomicAdd(&acc->payload[A * 4 + TOAST_AG], (unsigned long long)size);
                  atomicAdd(&acc->count[A * 4 + TOAST_AG], 1u);
                  size *= (uint64_t)T.sizes[A];
                }
              }
              for (int A = 0; A < T.n_axes; ++A) {          // phase 2: RS / AR
                if (!((P >> A) & 1)) continue;
                if (dim_of(U, A) >= 0) {
                  size = exdiv(T, size, 1u << A);
                  atomicAdd(&acc->payload[A * 4 + TOAST_RS], (unsigned long long)size);
                  atomicAdd(&acc->count[A * 4 + TOAST_RS], 1u);
                } else {
                  atomicAdd(&acc->payload[A * 4 + TOAST_AR], (unsigned long long)size);
                  atomicAdd(&acc->count[A * 4 + TOAST_AR], 1u);
                }
              }
              gk[k] = (long long)exdiv(T, dop.gbytes, Up) - (long long)exdiv(T, dop.gbytes, Dp);
            }
          }
        }
      }
      // temporaries: per distinct operand value, the largest growth (C11/C12)
#pragma unroll
      for (int k = 0; k < MAX_USES_PER_OP; ++k) {
        if (k < (int)op.n_uses) {
          bool first = true;
#pragma unroll
          for (int k2 = 0; k2 < k; ++k2) first &= (vk[k2] != vk[k]);
          if (first) {
            long long mx = 0;
#pragma unroll
            for (int k2 = k; k2 < MAX_USES_PER_OP; ++k2)
              if (vk[k2] == vk[k] && gk[k2] > mx) mx = gk[k2];
            temp_total += mx;
          }
        }
      }
      // values whose last use is this op (C12)
      long long dying = 0;
      for (uint32_t i = 0; i < op.n_death; ++i) {
        uint32_t v = __ldg(T.deaths + op.death_begin + i);
        if (v == (uint32_t)t) {
          dying += res;
        } else {
          OpRec vo = load_op(T, v);
          Mat vm = materialize(T, acol, vo.loop_begin, vo.n_loops, zr, on);
          dying += (long long)exdiv(T, vo.gbytes, dims_or(site_masks(vm.masks, vo.res_roles, vo.rank)));
        }
      }
      delta = res - dying;
      inop = res + temp_total;
    }
    // H5: warp inclusive scan of the live-byte deltas, then max of M_t
    long long incl = delta;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      long long y = __shfl_up_sync(FULL, incl, off);
      if (lane >= off) incl += y;
    }
    long long M = live ? carry + (incl - delta) + inop : LLONG_MIN;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      long long y = __shfl_xor_sync(FULL, M, off);
      M = y > M ? y : M;
    }
    if (M > peak) peak = M;
    carry += __shfl_sync(FULL, incl, 31);
  }
  // ---------------- reductions
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    key += __shfl_xor_sync(FULL, key, off);
    uint64_t olo = __shfl_xor_sync(FULL, flo, off), ohi = __shfl_xor_sync(FULL, fhi, off);
    uint64_t nlo = flo + olo;
    fhi = fhi + ohi + (nlo < flo ? 1 : 0);
    flo = nlo;
  }
  __syncwarp();
  // ---------------- H6 score (C13), fixed evaluation order, no FMA
  if (lane == 0) {
    double fl = __dadd_rn(__dmul_rn(__ull2double_rn(fhi), 18446744073709551616.0), __ull2double_rn(flo));
    double t = __ddiv_rn(fl, T.F);
    unsigned long long ncoll = 0;
    for (int A = 0; A < T.n_axes; ++A) {
      double n = (double)T.sizes[A];
      double ag = __ull2double_rn(acc->payload[A * 4 + 0]), rs = __ull2double_rn(acc->payload[A * 4 + 1]);
      double ar = __ull2double_rn(acc->payload[A * 4 + 2]), a2a = __ull2double_rn(acc->payload[A * 4 + 3]);
      double n1 = __dsub_rn(n, 1.0);
      double p1 = __dmul_rn(n1, __dadd_rn(ag, rs));
      double p2 = __ddiv_rn(__dmul_rn(n1, __dadd_rn(__dmul_rn(2.0, ar), a2a)), n);
      double term = __ddiv_rn(__dadd_rn(p1, p2), T.bw[A]);
      t = __dadd_rn(t, term);
    }
    uint64_t pk = (uint64_t)peak;
    double RT = __ddiv_rn(t, T.t0);
    double MP = pk > T.DM ? __ddiv_rn(__dmul_rn(T.C, __ull2double_rn(pk - T.DM)), __ull2double_rn(T.peak0)) : 0.0;
    double score = __dadd_rn(RT, MP);
    toast_cost* c = reinterpret_cast<toast_cost*>(rec);
    memset(c, 0, sizeof(toast_cost));
    c->runtime_s = t;
    c->score = score;
    c->peak_bytes = pk;
    c->flops = flo;
    c->flops_hi = fhi;
    c->state_key = key;
    c->status = 0;
    for (int q = 0; q < 16; ++q) {
      unsigned int cq = acc->count[q];
      ncoll += cq;
      c->payload[q >> 2][q & 3] = acc->payload[q];
      c->count[q >> 2][q & 3] = (uint16_t)(cq > 65535u ? 65535u : cq);
    }
    c->n_collectives = (uint32_t)ncoll;
  }
  __syncwarp();
  reinterpret_cast<unsigned long long*>(out)[lane] = rec[lane];
  if (ok) acol[ac] = 0u;   // restore the all-zero invariant for the next candidate
  __syncwarp();
}

struct WarpSmem {
  uint32_t* acol;
  Acc* acc;
  unsigned long long* rec;
};

__device__ __forceinline__ WarpSmem warp_smem(int n_acolors) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const int acol_bytes = ((n_acolors * 4) + 15) & ~15;
  const int per = acol_bytes + (int)sizeof(Acc) + 256;
  unsigned char* base = smem + (size_t)warp * per;
  WarpSmem w;
  w.rec = reinterpret_cast<unsigned long long*>(base);
  w.acc = reinterpret_cast<Acc*>(base + 256);
  w.acol = reinterpret_cast<uint32_t*>(base + 256 + sizeof(Acc));
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < n_acolors; i += 32) w.acol[i] = 0u;
  __syncwarp();
  return w;
}

__global__ void __launch_bounds__(256) toast_eval_kernel(const DeviceTables T, const uint16_t* __restrict__ seqs,
                                                         int64_t n, toast_cost* __restrict__ out) {
  WarpSmem w = warp_smem(T.n_acolors);
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    uint32_t sid = seqs[i * 32 + lane];
    eval_warp(T, sid, w.acol, w.acc, w.rec, out + i);
  }
}

// ---------------- K2: rollouts (C15)
__device__ __forceinline__ void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                              uint32_t k1, uint32_t& o0, uint32_t& o1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  o0 = c0;
  o1 = c1;
}

__global__ void __launch_bounds__(256) toast_rollout_kernel(const DeviceTables T, const uint16_t* __restrict__ pre,
                                                            int64_t n, uint64_t seed, uint64_t id_base,
                                                            uint16_t* __restrict__ out_seqs,
                                                            toast_cost* __restrict__ out) {
  WarpSmem w = warp_smem(T.n_acolors);
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const uint32_t seed_lo = (uint32_t)seed, seed_hi = (uint32_t)(seed >> 32);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    uint32_t p = pre[i * 32 + lane];
    unsigned zb = __ballot_sync(FULL, p == 0);
    int stop = zb ? __ffs(zb) - 1 : 32;
    bool bad = __ballot_sync(FULL, (lane > stop && p != 0) || (lane < stop && (int)p >= T.n_actions)) != 0;
    uint32_t sv = p;
    if (!bad) {
      uint32_t legal = 0;
      if (lane < T.n_words) {
        legal = FULL;
        int hi = T.n_actions - lane * 32;   // ids >= n_actions are not actions
        if (hi < 32) legal = hi <= 0 ? 0u : ((1u << hi) - 1u);
        if (lane == 0) legal &= ~1u;        // STOP is not in the legal set
      }
      for (int j = 0; j < stop; ++j) {
        uint32_t a = __shfl_sync(FULL, p, j);
        if (lane < T.n_words) legal &= ~__ldg(T.kill + (size_t)a * T.n_words + lane);
      }
      const uint64_t id = id_base + (uint64_t)i;
      for (int d = stop; d < T.max_depth; ++d) {
        uint32_t r0, r1;
        philox4x32_10((uint32_t)id, (uint32_t)(id >> 32), (uint32_t)d, 0u, seed_lo, seed_hi, r0, r1);
        if ((uint64_t)r0 * (uint64_t)T.max_depth < ((uint64_t)d << 32)) break;   // p_stop = d / max_depth
        uint32_t cnt = __popc(legal);
        uint32_t incl = cnt;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          uint32_t y = __shfl_up_sync(FULL, incl, off);
          if (lane >= off) incl += y;
        }
        uint32_t total = __shfl_sync(FULL, incl, 31);
        if (total == 0) break;
        uint32_t k = (uint32_t)(((uint64_t)r1 * total) >> 32);
        uint32_t excl = incl - cnt;
        bool own = k >= excl && k < incl;
        int owner = __ffs(__ballot_sync(FULL, own)) - 1;
        uint32_t a = 0;
        if (own) {
          uint32_t wv = legal;
          for (uint32_t q = excl; q < k; ++q) wv &= wv - 1;
          a = (uint32_t)lane * 32 + (uint32_t)(__ffs(wv) - 1);
        }
        a = __shfl_sync(FULL, a, owner);
        if (lane < T.n_words) legal &= ~__ldg(T.kill + (size_t)a * T.n_words + lane);
        if (lane == d) sv = a;
      }
    }
    out_seqs[i * 32 + lane] = (uint16_t)sv;
    eval_warp(T, sv, w.acol, w.acc, w.rec, out + i);
  }
}

int smem_per_warp(int n_acolors) { return (((n_acolors * 4) + 15) & ~15) + (int)sizeof(Acc) + 256; }

}  // namespace

// ============================================================== host side
bool is_device_pointer(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

#define TOAST_CUDA(call)                                                              \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      err = std::string(#call) + ": " + cudaGetErrorString(e_);                        \
      return e_ == cudaErrorMemoryAllocation ? TOAST_E_OOM : TOAST_E_CUDA;             \
    }                                                                                 \
  } while (0)

template <typename V>
static toast_status upload(toast_analysis* a, const V& v, const typename V::value_type** dst, std::string& err) {
  size_t bytes = std::max<size_t>(v.size() * sizeof(typename V::value_type), 16);
  void* d = nullptr;
  TOAST_CUDA(cudaMalloc(&d, bytes));
  a->dev_allocs.push_back(d);
  if (!v.empty()) TOAST_CUDA(cudaMemcpy(d, v.data(), v.size() * sizeof(typename V::value_type), cudaMemcpyHostToDevice));
  *dst = reinterpret_cast<const typename V::value_type*>(d);
  return TOAST_OK;
}

toast_status upload_tables(toast_analysis* a, std::string& err) {
  TOAST_CUDA(cudaSetDevice(a->device));
  DeviceTables& T = a->dt;
  toast_status st;
  if ((st = upload(a, a->h_ops, &T.ops, err))) return st;
  if ((st = upload(a, a->h_gflops, &T.gflops, err))) return st;
  if ((st = upload(a, a->h_loops, &T.loops, err))) return st;
  if ((st = upload(a, a->h_uses, &T.uses, err))) return st;
  if ((st = upload(a, a->h_deaths, &T.deaths, err))) return st;
  if ((st = upload(a, a->h_desel, &T.desel, err))) return st;
  if ((st = upload(a, a->h_actions, &T.actions, err))) return st;
  if ((st = upload(a, a->h_acol_groups, &T.acol_groups, err))) return st;
  if ((st = upload(a, a->h_kill, &T.kill, err))) return st;
  a->smem_per_warp = smem_per_warp(T.n_acolors);
  const int smem = 8 * a->smem_per_warp;
  if (smem > 48 * 1024) {
    TOAST_CUDA(cudaFuncSetAttribute(toast_eval_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    TOAST_CUDA(cudaFuncSetAttribute(toast_rollout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  }
  int sms = 0, be = 0, br = 0;
  TOAST_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, a->device));
  TOAST_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&be, toast_eval_kernel, 256, smem));
  TOAST_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&br, toast_rollout_kernel, 256, smem));
  a->eval_blocks = sms * std::max(be, 1);
  a->rollout_blocks = sms * std::max(br, 1);
  return TOAST_OK;
}

void free_tables(toast_analysis* a) {
  if (a->device >= 0) cudaSetDevice(a->device);
  for (void* p : a->dev_allocs) cudaFree(p);
  a->dev_allocs.clear();
  if (a->scratch) cudaFree(a->scratch);
  a->scratch = nullptr;
  a->scratch_bytes = 0;
}

toast_status launch_eval(const toast_analysis* a, const uint16_t* d_seqs, int64_t n, toast_cost* d_out, void* stream,
                         std::string& err) {
  if (n <= 0) return TOAST_OK;
  int64_t blocks = std::min<int64_t>((n + 7) / 8, a->eval_blocks);
  toast_eval_kernel<<<(unsigned)blocks, 256, 8 * a->smem_per_warp, (cudaStream_t)stream>>>(a->dt, d_seqs, n, d_out);
  TOAST_CUDA(cudaGetLastError());
  return TOAST_OK;
}

toast_status launch_rollout(const toast_analysis* a, const uint16_t* d_pre, int64_t n, uint64_t seed, uint64_t id_base,
                            uint16_t* d_seqs, toast_cost* d_out, void* stream, std::string& err) {
  if (n <= 0) return TOAST_OK;
  int64_t blocks = std::min<int64_t>((n + 7) / 8, a->rollout_blocks);
  toast_rollout_kernel<<<(unsigned)blocks, 256, 8 * a->smem_per_warp, (cudaStream_t)stream>>>(a->dt, d_pre, n, seed,
                                                                                             id_base, d_seqs, d_out);
  TOAST_CUDA(cudaGetLastError());
  return TOAST_OK;
}

// host-pointer path: stage through device scratch on `stream`, then wait
toast_status run_host_buffers(toast_analysis* a, bool rollout, const uint16_t* h_in, int64_t n, uint64_t seed,
                              uint64_t id_base, uint16_t* h_seqs, toast_cost* h_out, void* stream, std::string& err) {
  if (n <= 0) return TOAST_OK;
  std::lock_guard<std::mutex> lk(a->scratch_mu);
  const size_t in_b = (size_t)n * 64, out_b = (size_t)n * sizeof(toast_cost);
  const size_t need = out_b + in_b + (rollout ? in_b : 0);
  if (a->scratch_bytes < need) {
    if (a->scratch) cudaFree(a->scratch);
    a->scratch = nullptr;
    a->scratch_bytes = 0;
    TOAST_CUDA(cudaMalloc(&a->scratch, need));
    a->scratch_bytes = need;
  }
  cudaStream_t s = (cudaStream_t)stream;
  toast_cost* d_out = reinterpret_cast<toast_cost*>(a->scratch);
  uint16_t* d_in = reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(a->scratch) + out_b);
  uint16_t* d_seqs = reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(a->scratch) + out_b + in_b);
  TOAST_CUDA(cudaMemcpyAsync(d_in, h_in, in_b, cudaMemcpyHostToDevice, s));
  toast_status st = rollout ? launch_rollout(a, d_in, n, seed, id_base, d_seqs, d_out, stream, err)
                            : launch_eval(a, d_in, n, d_out, stream, err);
  if (st) return st;
  TOAST_CUDA(cudaMemcpyAsync(h_out, d_out, out_b, cudaMemcpyDeviceToHost, s));
  if (rollout) TOAST_CUDA(cudaMemcpyAsync(h_seqs, d_seqs, in_b, cudaMemcpyDeviceToHost, s));
  TOAST_CUDA(cudaStreamSynchronize(s));
  return TOAST_OK;
}

}  // namespace toast
