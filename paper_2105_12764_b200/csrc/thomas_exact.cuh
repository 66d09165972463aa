// thomas_exact.cuh -- exact-policy batched Thomas solve with the fibers
// resident in shared memory: one HBM read and one HBM write per element.
//
// The recurrence (thomas_fiber, kernels.hpp:143-151) is evaluated in the
// reference's order with the _rn intrinsics, one lane per fiber, so results
// are bit-identical to the reference.  A CTA stages the tile of NF fibers
// with asynchronous copies by all its threads (the same position-major /
// row-major layouts as thomas_fiber.cuh), one warp runs the NF sequential
// recurrences out of shared memory, and all threads write the solution (or
// the fused epilogue of the level's last solve) back with coalesced stores.
// Several CTAs per SM overlap one CTA's recurrence with the others' copies.
#pragma once

#include "common.cuh"
#include "level.cuh"
#include "thomas_fiber.cuh"

namespace mgrg {

constexpr int kTeThreads = 256;

template <typename R> __host__ __device__ constexpr int te_nf() {
  return sizeof(R) == 4 ? 32 : 16;
}
// tile elements: DIM 2 with 32 fibers stages 16-byte supersets of each row
template <typename R> __host__ __device__ inline size_t te_tile_elems(int dim, uint32_t m) {
  constexpr int v = 16 / int(sizeof(R));
  const size_t pitch = (te_nf<R>() == 32 && dim == 2) ? size_t((32 + 2 * v - 2) / v * v)
                                                      : size_t(te_nf<R>());
  return pitch * m;
}
template <typename R> __host__ __device__ inline size_t te_smem(int dim, uint32_t m) {
  return te_tile_elems<R>(dim, m) * sizeof(R);
}
// used when three CTAs fit on an SM (every 3-D level up to 1025^3)
template <typename R> inline bool te_fits(int dim, uint32_t m) {
  return m >= 2 && te_smem<R>(dim, m) <= 74 * 1024;
}

// DIM 0: fibers are rows along x; DIM 1: fiber F = x + m0 * z, position i at
// x + m0 * (i + m1 * z); DIM 2: fiber F = x + m0 * y, position i at F + m01 * i.
template <typename R, int DIM>
__global__ void __launch_bounds__(kTeThreads, 3)
    thomas_exact_kernel(R *f, ThomasGeom<R> t, uint64_t nfib, uint32_t m0, uint32_t m1,
                        Epi epi, const R *base, R *out) {
  pdl_wait();
  // f, base and out may alias (epilogues write in place)
  constexpr int NF = te_nf<R>();
  constexpr int V = 16 / int(sizeof(R));
  constexpr int NCK = (NF + 2 * V - 2) / V; // 16-byte chunks of a row superset
  constexpr int RW = NCK * V;
  constexpr bool SUP = DIM == 2 && NF == 32;
  extern __shared__ __align__(16) unsigned char te_raw[];
  R *tile = reinterpret_cast<R *>(te_raw);
  const uint32_t m = t.m;
  const int tid = threadIdx.x;
  const uint64_t F0 = uint64_t(blockIdx.x) * NF;
  const int nf = int(nfib - F0 < uint64_t(NF) ? nfib - F0 : uint64_t(NF));
  const uint64_t m01 = uint64_t(m0) * m1;
  const uint64_t ps = DIM == 1 ? m0 : m01; // position stride (DIM 1, 2)
  const uint64_t ntot = nfib * m;
  // the thread's fiber is fixed (kTeThreads is a multiple of NF): its
  // address once, then running pointers along the positions
  static_assert(kTeThreads % NF == 0, "thread -> fiber map");
  constexpr int PSTEP = kTeThreads / NF; // positions per pass of the CTA
  const int my_fi = tid % NF;
  const uint32_t my_i0 = uint32_t(tid / NF);
  uint64_t fa;
  {
    const uint64_t F = F0 + uint64_t(my_fi < nf ? my_fi : nf - 1);
    fa = DIM == 1 ? (F % m0) + m01 * (F / m0) : F;
  }
  // superset row shift of position i: (F0 + ps * i) mod V in 32 bits
  const uint32_t sh0 = uint32_t(F0) & (V - 1), shp = uint32_t(ps) & (V - 1);
  auto shift = [&](uint32_t i) { return (sh0 + shp * i) & uint32_t(V - 1); };

  // ---- stage
  if (DIM == 0) {
    const R *src = f + F0 * m;
    const uint32_t n = uint32_t(nf) * m, nv = n / V;
    for (uint32_t e = tid; e < nv; e += kTeThreads)
      cp_async16(tile + e * V, src + e * V);
    for (uint32_t e = nv * V + tid; e < n; e += kTeThreads)
      cp_async(tile + e, src + e);
  } else if (SUP) {
    for (uint32_t e = tid; e < m * NCK; e += kTeThreads) {
      const uint32_t i = e / NCK, c = e % NCK;
      const uint64_t g = ((F0 + ps * i) & ~uint64_t(V - 1)) + uint64_t(c) * V;
      R *d = tile + size_t(i) * RW + c * V;
      if (g + V <= ntot) {
        cp_async16(d, f + g);
      } else {
        for (int q = 0; q < V; ++q)
          if (g + q < ntot)
            cp_async(d + q, f + g + q);
      }
    }
  } else {
    const R *src = f + fa + ps * my_i0;
    for (uint32_t i = my_i0; i < m; i += PSTEP, src += ps * PSTEP)
      cp_async(tile + size_t(i) * NF + my_fi, src);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  // ---- one lane per fiber: forward elimination, back substitution
  if (tid < NF && tid < nf) {
    const int fi = tid;
    R *p;
    uint32_t st;
    if (DIM == 0) {
      p = tile + size_t(fi) * m;
      st = 1;
    } else {
      p = tile + fi;
      st = SUP ? RW : NF;
    }
    auto at = [&](uint32_t i) -> R & {
      if constexpr (SUP)
        return p[size_t(i) * st + shift(i)];
      else
        return p[size_t(i) * st];
    };
    const R *fwd = t.fwd, *ip = t.ip, *h = t.h;
    // blocks of B positions: the tile and factor loads of a block are
    // independent of the recurrence and issue together; only the mul/add
    // chain is sequential
    constexpr int B = 8;
    R prev = at(0);
    uint32_t i = 1;
    for (; i + B <= m; i += B) {
      R v[B], a[B];
#pragma unroll
      for (int k = 0; k < B; ++k) {
        v[k] = at(i + k);
        a[k] = __ldg(fwd + i + k);
      }
#pragma unroll
      for (int k = 0; k < B; ++k) {
        prev = add(v[k], mul(a[k], prev));
        v[k] = prev;
      }
#pragma unroll
      for (int k = 0; k < B; ++k)
        at(i + k) = v[k];
    }
    for (; i < m; ++i) {
      prev = add(at(i), mul(__ldg(fwd + i), prev));
      at(i) = prev;
    }
    R next = mul(prev, __ldg(ip + m - 1));
    at(m - 1) = next;
    int j = int(m) - 2; // descending positions m-2 .. 0
    for (; j + 1 >= B; j -= B) {
      R v[B], hh[B], pp[B];
#pragma unroll
      for (int k = 0; k < B; ++k) {
        v[k] = at(uint32_t(j - k));
        hh[k] = __ldg(h + j - k);
        pp[k] = __ldg(ip + j - k);
      }
#pragma unroll
      for (int k = 0; k < B; ++k) {
        next = mul(sub(v[k], mul(hh[k], next)), pp[k]);
        v[k] = next;
      }
#pragma unroll
      for (int k = 0; k < B; ++k)
        at(uint32_t(j - k)) = v[k];
    }
    for (; j >= 0; --j) {
      next = mul(sub(at(uint32_t(j)), mul(__ldg(h + j), next)), __ldg(ip + j));
      at(uint32_t(j)) = next;
    }
  }
  __syncthreads();

  // ---- write back (epilogue of the level's last solve)
  auto emit = [&](uint64_t gidx, R z) {
    if (epi == Epi::none)
      f[gidx] = z;
    else
      out[gidx] = epi == Epi::add ? add(base[gidx], z) : sub(base[gidx], z);
  };
  if (DIM == 0) {
    const uint32_t n = uint32_t(nf) * m;
    for (uint32_t e = tid; e < n; e += kTeThreads)
      emit(F0 * m + e, tile[e]);
  } else if (my_fi < nf) {
    uint64_t gi = fa + ps * my_i0;
    for (uint32_t i = my_i0; i < m; i += PSTEP, gi += ps * PSTEP) {
      const R z = SUP ? tile[size_t(i) * RW + shift(i) + my_fi] : tile[size_t(i) * NF + my_fi];
      emit(gi, z);
    }
  }
}

} // namespace mgrg
