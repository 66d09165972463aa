// thomas_fiber.cuh -- FAST-policy batched Thomas solve with whole fibers
// resident on chip: one HBM read and one HBM write per element.
//
// The level-(l-1) mass matrix along a dimension is the same for every fiber
// (TridiagonalOperator::build, kernels.hpp:98-136), so the recurrences
//   forward : v_i = f_i + fwd_i * v_{i-1}
//   backward: x_i = ip_i * v_i + g_i * x_{i+1},   g_i = -ip_i * h_i
// (thomas_fiber, kernels.hpp:143-151, rearranged: same operator) split into
// chunks with fiber-independent carry maps: a chunk [a, b) solved with a
// zero carry-in is corrected by PF_i * c (forward, PF_i = prod_{a..i} fwd)
// and PB_i * d (backward, PB_i = prod_{i..b-1} g), where the carries c, d
// follow from the neighbouring chunks' end values by a short sequential
// pass over the 16 chunks of the CTA (host-precomputed chunk multipliers).
//
// CTA = 32 fibers x 16 chunks: warp w owns chunk w of every fiber, lane =
// fiber, and keeps the chunk (<= CH values) in registers through all three
// passes.  The tile is staged through shared memory with asynchronous
// copies (no registers held by loads in flight): y/z fibers as [position]
// [fiber] rows (position i of the 32 fibers is a row of 32 consecutive x
// nodes, coalesced), x fibers as the contiguous region of 32 rows with
// 16-byte copies (pitch m, odd on dyadic levels: conflict-free per-fiber
// reads).  y/z results go straight to HBM per position; x results back
// through the tile with 16-byte stores.  The last solve of a
// level fuses the epilogue (a_{l-1} = P + z on decompose, coarse' =
// a_{l-1} - z on recompose).
#pragma once

#include <type_traits>

#include "common.cuh"
#include "level.cuh"

namespace mgrg {

constexpr int kTfThreads = 512; // threads per CTA = fibers x chunks

// Fiber-group shape for a fiber length m: NF fibers x NCH = 512/NF chunks
// per CTA with chunks of at most 33 positions.  Short fibers (m <= 528,
// every 3-D level here) use 32 fibers per CTA (a warp = one chunk of 32
// fibers: coalesced position rows); long 2-D fibers (m <= 4224) 4 fibers
// x 128 chunks.  0 = not handled (the streaming kernels take over).
__host__ __device__ inline int tf_nf(uint32_t m) {
  return m <= 16u * 33u ? 32 : (m <= 128u * 33u ? 4 : 0);
}
__host__ __device__ inline int tf_nch(uint32_t m) {
  const int nf = tf_nf(m);
  return nf ? kTfThreads / nf : 0;
}

// Tables: q8[i] = {fwd_i, ip_i, g_i, PF_i, PB_i, 0, 0, 0}, then the chunk
// multipliers pfend[w] (PF at the chunk end), pbstart[w] (PB at its start),
// w < tf_nch(m).
template <typename R> struct ThomasLean {
  const R *tab; // [8m] q8, [nch] pfend, [nch] pbstart
  uint32_t m;
};
// chunk length of a fiber length (the kernel instantiation), 0 = not handled
__host__ __device__ inline int tf_ch(uint32_t m) {
  const int nch = tf_nch(m);
  if (!nch)
    return 0;
  const uint32_t c = (m + nch - 1) / nch;
  const int cls[7] = {1, 2, 3, 5, 9, 17, 33};
  for (int i = 0; i < 7; ++i)
    if (c <= uint32_t(cls[i]))
      return cls[i];
  return 0;
}
// positions covered by the chunks (every chunk exactly CH long; positions
// m .. mp-1 are padding: fwd = g = 0, so they decouple and solve to 0)
__host__ __device__ inline uint32_t tf_padded(uint32_t m) {
  return uint32_t(tf_nch(m)) * uint32_t(tf_ch(m));
}
template <typename R> __host__ __device__ inline size_t tf_tab_elems(uint32_t m) {
  return 8 * size_t(tf_padded(m) > m ? tf_padded(m) : m) + 2 * size_t(tf_nch(m));
}
// the coefficient table is staged in shared memory when it fits beside the
// tile (every 3-D level); long 2-D fibers read it through L1
template <typename R> __host__ __device__ inline bool tf_tab_smem(uint32_t m) {
  return tf_nf(m) == 32;
}
// shared memory: [tile NF x m][carries NCH x NF][tables], 16-byte aligned parts
template <typename R> __host__ __device__ inline size_t tf_tile_elems(int dim, uint32_t m) {
  // NF fibers per position; z fibers in 32-fiber groups are staged with
  // 16-byte chunks of a superset (pitch (32 + 2V - 2) / V * V, V = 16/sizeof(R))
  const int nf = tf_nf(m), v = 16 / int(sizeof(R));
  const size_t pitch =
      (nf == 32 && dim == 2) ? size_t((32 + 2 * v - 2) / v * v) : size_t(nf);
  return (pitch * m + 3) & ~size_t(3);
}
template <typename R> __host__ __device__ inline size_t tf_smem(int dim, uint32_t m) {
  return (tf_tile_elems<R>(dim, m) + size_t(kTfThreads) +
          (tf_tab_smem<R>(m) ? tf_tab_elems<R>(m) : 0)) *
         sizeof(R);
}

// 16-byte async copy of n elements (src, dst 16-byte aligned) by the CTA.
template <typename R>
__device__ __forceinline__ void tf_copy_in(R *dst, const R *src, uint32_t n, int tid) {
  constexpr int V = 16 / sizeof(R);
  const uint32_t nv = n / V;
  for (uint32_t e = tid; e < nv; e += kTfThreads)
    cp_async16(dst + e * V, src + e * V);
  for (uint32_t e = nv * V + tid; e < n; e += kTfThreads)
    cp_async(dst + e, src + e);
}

// DIM 0: fibers are rows along x (fiber id = row id, positions contiguous);
// DIM 1: fiber id F = x + m0 * z, position i at x + m0 * (i + m1 * z);
// DIM 2: fiber id F = x + m0 * y, position i at F + m0 * m1 * i.
// Thread t: fiber t % NF, chunk t / NF.
template <typename R, int DIM, int CH, int NF>
__global__ void __launch_bounds__(kTfThreads, sizeof(R) == 4 ? 2 : 1)
    thomas_fiber_kernel(R *__restrict__ f, ThomasLean<R> t, uint64_t nfib, uint32_t m0,
                        uint32_t m1, Epi epi, const R *base, R *out) {
  pdl_wait();
  constexpr int NCH = kTfThreads / NF;
  constexpr bool TSM = NF == 32; // coefficient table in shared memory
  extern __shared__ __align__(16) unsigned char tf_raw[];
  R *sm = reinterpret_cast<R *>(tf_raw);
  const uint32_t m = t.m;
  R *tile = sm;
  R *carry = sm + tf_tile_elems<R>(DIM, m);
  R *stab = carry + kTfThreads;
  const R *tab = TSM ? stab : t.tab;
  const uint32_t mp = uint32_t(NCH) * CH; // padded positions (>= m)
  const R *pfend = tab + 8 * size_t(mp > m ? mp : m), *pbstart = pfend + NCH;
  const int tid = threadIdx.x, fi = tid % NF, w = tid / NF;
  const uint64_t F0 = uint64_t(blockIdx.x) * NF;
  const int nf = int(nfib - F0 < uint64_t(NF) ? nfib - F0 : uint64_t(NF));
  const uint64_t m01 = uint64_t(m0) * m1;
  // chunk w = [a, a + CH); real positions a .. a + len - 1 (len <= CH)
  const uint32_t a = uint32_t(w) * CH;
  const uint32_t len = a >= m ? 0u : (m - a < uint32_t(CH) ? m - a : uint32_t(CH));

  // fiber address of the thread (DIM 1, 2; fibers past the end repeat the last)
  uint64_t fa = 0;
  if (DIM == 1) {
    const uint64_t F = F0 + min(fi, nf - 1);
    fa = (F % m0) + m01 * (F / m0);
  } else if (DIM == 2) {
    fa = F0 + min(fi, nf - 1);
  }
  const uint64_t ps = DIM == 1 ? m0 : m01; // position stride (DIM 1, 2)
  // 16-byte staging of whole position rows (DIM 1, 2 with 32 fibers): the
  // CTA's fibers must be one contiguous run of x nodes (DIM 1: not across a
  // z plane; DIM 2: always)
  constexpr int V = 16 / int(sizeof(R));
  constexpr int NCK = (NF + 2 * V - 2) / V; // chunks of a row superset
  constexpr int RW = NCK * V;               // staged row pitch (elements)
  const uint64_t F0row = DIM == 1 ? (F0 % m0) + m01 * (F0 / m0) : F0;
  const bool contiguous = DIM == 2 || (F0 % m0) + uint64_t(nf) <= m0;
  const uint64_t ntot = nfib * m;

  // DIM 1, 2: position-major tile [i][fiber]; with 32 contiguous fibers of
  // DIM 2 each position row is fetched as its 16-byte aligned superset (NCK
  // chunks, one LDGSTS.128 each: ~4x fewer copy operations than element
  // copies) and read back at the row's shift.  The same staging brings the
  // epilogue's base rows in while the solve runs.
  constexpr bool SUPR = NF == 32 && DIM == 2;
  auto stage_rows = [&](const R *src) {
    if (SUPR && contiguous) {
      constexpr int RPR = 32 / NCK; // rows per warp copy instruction
      const int lane = tid & 31;
      for (uint32_t i0 = w; i0 < m; i0 += NCH * RPR) {
        const uint32_t i = i0 + uint32_t(lane / NCK) * NCH;
        const int c = lane % NCK;
        if (lane < RPR * NCK && i < m) {
          const uint64_t s0 = (F0row + ps * i) & ~uint64_t(V - 1);
          const uint64_t g = s0 + uint64_t(c) * V;
          R *d = tile + size_t(i) * RW + c * V;
          if (g + V <= ntot) {
            cp_async16(d, src + g);
          } else {
#pragma unroll
            for (int e = 0; e < V; ++e)
              if (g + e < ntot)
                cp_async(d + e, src + g + e);
          }
        }
      }
    } else {
      for (uint32_t i = w; i < m; i += NCH)
        cp_async(tile + size_t(i) * NF + fi, src + fa + ps * i);
    }
  };
  auto row_at = [&](uint32_t i) -> R {
    if (SUPR && contiguous)
      return tile[size_t(i) * RW + int((F0row + ps * i) & uint64_t(V - 1)) + fi];
    return tile[size_t(i) * NF + fi];
  };

  if (TSM)
    tf_copy_in(stab, t.tab, tf_tab_elems<R>(m), tid);
  R v[CH];
  if (DIM == 0) {
    tf_copy_in(tile, f + F0 * m, uint32_t(nf) * m, tid);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    const uint32_t ln = fi < nf ? len : 0u;
    const R *tp = tile + uint32_t(fi) * m + a;
#pragma unroll
    for (int k = 0; k < CH; ++k)
      v[k] = uint32_t(k) < ln ? tp[k] : R(0);
  } else {
    stage_rows(f);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
#pragma unroll
    for (int k = 0; k < CH; ++k)
      v[k] = uint32_t(k) < len ? row_at(a + k) : R(0);
  }

  // ---- forward, zero carry-in
  R acc = R(0);
  const R *qa = tab + 8 * size_t(a);
#pragma unroll
  for (int k = 0; k < CH; ++k) { // padded positions: fwd = 0, v = 0
    acc = fma(qa[8 * k], acc, v[k]);
    v[k] = acc;
  }
  carry[w * NF + fi] = acc;
  __syncthreads(); // every thread has read its tile values
  const bool pre = DIM != 0 && epi != Epi::none;
  if (pre) { // the epilogue's base rows, in flight during the solve
    stage_rows(base);
    cp_async_commit();
  }
  R c = R(0);
  for (int k = 0; k < w; ++k)
    c = fma(pfend[k], c, carry[k * NF + fi]);
  // ---- forward fix-up + backward, zero carry-in (descending)
  R x = R(0);
#pragma unroll
  for (int k = CH - 1; k >= 0; --k) { // padded positions: g = 0, x = ip * v
    const R *q = qa + 8 * k;
    const R vj = fma(q[3], c, v[k]);
    x = fma(q[2], x, q[1] * vj);
    v[k] = x;
  }
  __syncthreads(); // every thread has read the forward carries
  carry[w * NF + fi] = x;
  __syncthreads();
  R d = R(0);
  for (int k = NCH - 1; k > w; --k)
    d = fma(pbstart[k], d, carry[k * NF + fi]);
  // ---- backward fix-up, epilogue, store
#pragma unroll
  for (int k = 0; k < CH; ++k)
    v[k] = fma(qa[8 * k + 4], d, v[k]);
  if (DIM == 0) {
    if (fi < nf) {
      R *tq = tile + uint32_t(fi) * m + a;
#pragma unroll
      for (int k = 0; k < CH; ++k)
        if (uint32_t(k) < len)
          tq[k] = v[k];
    }
    __syncthreads();
    constexpr int V = 16 / sizeof(R);
    using VT = typename std::conditional<sizeof(R) == 4, float4, double2>::type;
    const uint32_t n = uint32_t(nf) * m, nv = n / V;
    R *dst = epi == Epi::none ? f + F0 * m : out + F0 * m;
    const R *bs = base + F0 * m;
    const bool vec = ((reinterpret_cast<uintptr_t>(dst) |
                       (epi == Epi::none ? 0 : reinterpret_cast<uintptr_t>(bs))) & 15) == 0;
    for (uint32_t e = vec ? uint32_t(tid) : nv; e < nv; e += kTfThreads) {
      VT z = *reinterpret_cast<const VT *>(tile + e * V);
      if (epi != Epi::none) {
        const VT b = *reinterpret_cast<const VT *>(bs + e * V);
        R *zz = reinterpret_cast<R *>(&z);
        const R *bb = reinterpret_cast<const R *>(&b);
#pragma unroll
        for (int q = 0; q < V; ++q)
          zz[q] = epi == Epi::add ? bb[q] + zz[q] : bb[q] - zz[q];
      }
      *reinterpret_cast<VT *>(dst + e * V) = z;
    }
    for (uint32_t e = (vec ? nv * V : 0u) + tid; e < n; e += kTfThreads) {
      const R z = tile[e];
      dst[e] = epi == Epi::none ? z : (epi == Epi::add ? bs[e] + z : bs[e] - z);
    }
  } else {
    if (pre) {
      cp_async_wait<0>();
      __syncthreads();
    }
    if (fi < nf) {
      R *p = (epi == Epi::none ? f : out) + fa + ps * a;
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        if (uint32_t(k) < len) {
          if (epi == Epi::none) {
            *p = v[k];
          } else {
            const R b = row_at(a + k);
            *p = epi == Epi::add ? b + v[k] : b - v[k];
          }
        }
        p += ps;
      }
    }
  }
}

} // namespace mgrg

namespace mgrg {

// Small coarse lattices (the bottom levels of the hierarchy): all three
// solves of a level and the epilogue in ONE launch of one CTA, the lattice
// resident in shared memory.  Saves two launches per level on levels whose
// kernels are launch/latency bound (a few microseconds of work each).
// FAST policy; sequential Thomas per fiber (thomas_fiber, kernels.hpp:143-151)
// with the working-precision factors of TridiagonalOperator::build.
constexpr int kTsThreads = 512;
template <typename R> __host__ __device__ inline size_t ts_smem(uint64_t n, uint64_t ext_sum) {
  return size_t(n + 3 * ext_sum) * sizeof(R); // lattice + factors of every dim
}

template <typename R>
__global__ void __launch_bounds__(kTsThreads)
    thomas_small_kernel(R *__restrict__ f, ThomasGeom<R> tx, ThomasGeom<R> ty,
                        ThomasGeom<R> tz, uint32_t m0, uint32_t m1, uint32_t m2,
                        uint32_t refine, Epi epi, const R *base, R *out) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char ts_raw[];
  R *s = reinterpret_cast<R *>(ts_raw);
  const uint32_t n = m0 * m1 * m2;
  // the factors of every dimension go to shared memory with the lattice:
  // the recurrences below then never wait on a global load
  R *fac = s + n; // [d][fwd | ip | h] x m_d
  const uint32_t ext[3] = {m0, m1, m2};
  const uint32_t str[3] = {1, m0, m0 * m1};
  const ThomasGeom<R> *tg[3] = {&tx, &ty, &tz};
  uint32_t fo[3], acc = 0;
  for (int d = 0; d < 3; ++d) {
    fo[d] = acc;
    if ((refine >> d) & 1u)
      acc += 3 * ext[d];
  }
  for (uint32_t i = threadIdx.x; i < n; i += kTsThreads)
    s[i] = f[i];
  for (int d = 0; d < 3; ++d) {
    if (!((refine >> d) & 1u))
      continue;
    const uint32_t m = ext[d];
    for (uint32_t i = threadIdx.x; i < m; i += kTsThreads) {
      fac[fo[d] + i] = tg[d]->fwd[i];
      fac[fo[d] + m + i] = tg[d]->ip[i];
      fac[fo[d] + 2 * m + i] = i + 1 < m ? tg[d]->h[i] : R(0);
    }
  }
  __syncthreads();
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    if (!((refine >> d) & 1u))
      continue;
    const uint32_t m = ext[d], st = str[d], nf = n / m;
    const R *fw = fac + fo[d], *ip = fw + m, *hh = ip + m;
    for (uint32_t fb = threadIdx.x; fb < nf; fb += kTsThreads) {
      // fiber fb: position 0 at (fb % st) + (fb / st) * st * m
      R *p = s + (fb % st) + (fb / st) * st * m;
      R v = p[0];
      for (uint32_t i = 1; i < m; ++i) {
        v = fma(fw[i], v, p[i * st]);
        p[i * st] = v;
      }
      R x = v * ip[m - 1];
      p[(m - 1) * st] = x;
      for (uint32_t i = m - 1; i > 0; --i) {
        const uint32_t j = i - 1;
        x = (p[j * st] - hh[j] * x) * ip[j];
        p[j * st] = x;
      }
    }
    __syncthreads();
  }
  for (uint32_t i = threadIdx.x; i < n; i += kTsThreads) {
    const R z = s[i];
    if (epi == Epi::none)
      f[i] = z;
    else if (epi == Epi::add)
      out[i] = base[i] + z;
    else
      out[i] = base[i] - z;
  }
}

} // namespace mgrg
