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

// Fiber-group shape for a fiber length m: 32 fibers per CTA (a warp = one
// chunk of 32 fibers: coalesced position rows), tf_nw(m) chunks of at most
// 33 positions per CTA.  16-warp CTAs by default; f64 fibers of 73..2112
// positions use 8-warp CTAs (33 doubles per thread fill 128 registers, so a
// 16-warp CTA is alone on its SM and its load, solve and store phases never
// overlap; two 8-warp CTAs per SM do).  Fibers longer than one CTA's
// tf_nw x 33 positions (the long 2-D levels, e.g. 8193^2) are spread over a
// thread-block cluster of tf_cl(m) = 2, 4 or 8 CTAs, each holding a segment
// of the same 32 fibers, with the chunk carries exchanged through
// distributed shared memory (thomas_cluster_kernel).  0 = not handled (the
// streaming kernels take over).
#ifndef TF_NW8_F64
#define TF_NW8_F64 1
#endif
#ifndef TF_NW8_F32
#define TF_NW8_F32 0
#endif
// TF_CL16: 8-warp CTAs in non-portable 16-CTA clusters for f64 y / z fibers
// up to 4224 positions (else 16-warp CTAs in 8-CTA clusters there)
#ifndef TF_CL16
#define TF_CL16 0
#endif
template <typename R> __host__ __device__ inline int tf_maxcl(int nw) {
  return (TF_CL16 && sizeof(R) == 8 && nw == 8) ? 16 : 8;
}
template <typename R> __host__ __device__ inline int tf_nw(uint32_t m, int dim) {
  const bool on = sizeof(R) == 8 ? TF_NW8_F64 : TF_NW8_F32;
  return (on && dim != 0 && m > 8u * 9u && m <= 8u * 33u * uint32_t(tf_maxcl<R>(8))) ? 8 : 16;
}
template <typename R> __host__ __device__ inline int tf_cl(uint32_t m, int dim) {
  const int nw = tf_nw<R>(m, dim);
  const uint32_t seg = uint32_t(nw) * 33u;
  for (int cl = 1; cl <= tf_maxcl<R>(nw); cl *= 2)
    if (m <= seg * uint32_t(cl))
      return cl;
  return 0;
}
template <typename R> __host__ __device__ inline int tf_nf(uint32_t m, int dim) {
  return tf_cl<R>(m, dim) ? 32 : 0;
}
template <typename R> __host__ __device__ inline int tf_nch(uint32_t m, int dim) {
  return tf_nw<R>(m, dim) * tf_cl<R>(m, dim);
}
// served by thomas_cluster_kernel (clusters or 8-warp CTAs), else by
// thomas_fiber_kernel (one 16-warp CTA per fiber group)
template <typename R> __host__ __device__ inline bool tf_clustered(uint32_t m, int dim) {
  return tf_cl<R>(m, dim) > 1 || tf_nw<R>(m, dim) == 8;
}

// Tables: q8[i] = {fwd_i, ip_i, g_i, PF_i, PB_i, 0, 0, 0}, then the chunk
// multipliers pfend[w] (PF at the chunk end), pbstart[w] (PB at its start),
// w < tf_nch(m), then the cluster-segment multipliers mf[r] (product of the
// segment's pfend), mb[r] (product of its pbstart), r < tf_cl(m).
template <typename R> struct ThomasLean {
  const R *tab; // [8m] q8, [nch] pfend, [nch] pbstart
  uint32_t m;
};
// chunk length of a fiber length (the kernel instantiation), 0 = not handled
template <typename R> __host__ __device__ inline int tf_ch(uint32_t m, int dim) {
  const int nch = tf_nch<R>(m, dim);
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
template <typename R> __host__ __device__ inline uint32_t tf_padded(uint32_t m, int dim) {
  return uint32_t(tf_nch<R>(m, dim)) * uint32_t(tf_ch<R>(m, dim));
}
template <typename R> __host__ __device__ inline size_t tf_tab_elems(uint32_t m, int dim) {
  return 8 * size_t(tf_padded<R>(m, dim) > m ? tf_padded<R>(m, dim) : m) + 2 * size_t(tf_nch<R>(m, dim)) +
         2 * size_t(tf_cl<R>(m, dim));
}
// the coefficient table is staged in shared memory beside the tile
template <typename R> __host__ __device__ inline bool tf_tab_smem(uint32_t m, int dim) {
  return tf_nf<R>(m, dim) == 32;
}
// shared memory: [tile NF x m][carries NCH x NF][tables], 16-byte aligned parts
template <typename R> __host__ __device__ inline size_t tf_tile_elems(int dim, uint32_t m) {
  // NF fibers per position; y / z fibers in 32-fiber groups are staged with
  // 16-byte chunks of a superset (pitch (32 + 2V - 2) / V * V, V = 16/sizeof(R))
  const int nf = tf_nf<R>(m, dim), v = 16 / int(sizeof(R));
  const size_t pitch =
      (nf == 32 && dim != 0) ? size_t((32 + 2 * v - 2) / v * v) : size_t(nf);
  return (pitch * m + 3) & ~size_t(3);
}
template <typename R> __host__ __device__ inline size_t tf_smem(int dim, uint32_t m) {
  return (tf_tile_elems<R>(dim, m) + size_t(kTfThreads) +
          (tf_tab_smem<R>(m, dim) ? tf_tab_elems<R>(m, dim) : 0)) *
         sizeof(R);
}

// 16-byte async copy of n elements (src, dst 16-byte aligned) by the CTA.
template <typename R, int NT = kTfThreads>
__device__ __forceinline__ void tf_copy_in(R *dst, const R *src, uint32_t n, int tid) {
  constexpr int V = 16 / sizeof(R);
  const uint32_t nv = n / V;
  for (uint32_t e = tid; e < nv; e += NT)
    cp_async16(dst + e * V, src + e * V);
  for (uint32_t e = nv * V + tid; e < n; e += NT)
    cp_async(dst + e, src + e);
}

// DIM 0: fibers are rows along x (fiber id = row id, positions contiguous);
// DIM 1: fiber id F = x + m0 * z, position i at x + m0 * (i + m1 * z);
// DIM 2: fiber id F = x + m0 * y, position i at F + m0 * m1 * i.
// Thread t: fiber t % NF, chunk t / NF.
// CTAs per SM: x fibers of <= 17-position chunks run one more CTA per SM
// (measured at 1025^3 L9 f32 44.5 -> 37.9 us, 1025^2 x 513 L8 f64 46.7 ->
// 38.4 us; y / z fibers gain nothing and spill)
#ifndef TF_MINB_F32_SHORT
#define TF_MINB_F32_SHORT 3
#endif
#ifndef TF_MINB_F64_SHORT
#define TF_MINB_F64_SHORT 2
#endif
template <typename R, int DIM, int CH, int NF>
__global__ void __launch_bounds__(kTfThreads,
                                  sizeof(R) == 4 ? (DIM == 0 && CH <= 17 ? TF_MINB_F32_SHORT : 2)
                                                 : (DIM == 0 && CH <= 17 ? TF_MINB_F64_SHORT : 1))
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

  // DIM 1, 2: position-major tile [i][fiber]; with 32 contiguous fibers
  // each position row is fetched as its 16-byte aligned superset (NCK
  // chunks, one LDGSTS.128 each: ~4x fewer copy operations than element
  // copies) and read back at the row's shift.  The same staging brings the
  // epilogue's base rows in while the solve runs.
  constexpr bool SUPR = NF == 32 && DIM != 0;
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
    tf_copy_in(stab, t.tab, tf_tab_elems<R>(m, DIM), tid);
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

// ---- long fibers: thread-block clusters over 32-fiber groups -------------
//
// Fibers longer than one CTA's NW x 33 positions (tf_cl(m) = CL > 1) do not
// fit its registers: CTA r of a CL-CTA cluster holds positions
// [r*SEG, (r+1)*SEG), SEG = NW * CH, of a group of 32 fibers -- NW chunks in
// registers as in thomas_fiber_kernel -- so every element is still read once
// and written once.  The chunk carries of the sequential pass cross the
// segment boundaries through distributed shared memory: after its
// zero-carry-in pass every CTA publishes its segment's end value (forward:
// e_r, the value at the segment end; backward: b_r, at the segment start),
// the cluster barrier makes them visible, and CTA r composes the carry into
// its segment from its neighbours' published values with the
// host-precomputed segment multipliers mf / mb (c_{r+1} = mf_r * c_r + e_r;
// d_{r-1} = mb_r * d_r + b_r) before its own NW-chunk pass.  NW = 8 (f64,
// tf_nw) keeps two CTAs per SM; CL = 1 is the plain (cluster-free) case.
//
// A CTA holds (half) a register file of fiber values, so the kernel is
// persistent: the grid is the number of co-resident clusters,
// each cluster walks the fiber groups, and the shared-memory tile of the
// NEXT group is loaded (cp.async) as soon as the current group is in
// registers -- the load overlaps this group's solve, carry exchange and
// stores.  Results and epilogue bases go straight between registers and
// HBM (y / z fibers: position rows of 32 consecutive x nodes, coalesced;
// x fibers: each thread's chunk is a contiguous run, written sector by
// sector).  The segment's coefficient slice is staged once per CTA.
template <typename R, int DIM, int CH, int NW>
__host__ __device__ inline size_t tc_tile_elems() {
  constexpr size_t SEG = size_t(NW) * CH;
  return ((DIM == 0 ? 32 * (SEG + 1) : SEG * 32) + 3) & ~size_t(3);
}
// x fibers: per-warp output staging, 32 fibers x 8 positions (pitch 9)
constexpr int kTcStg = 32 * 9;
template <typename R, int DIM, int CH, int NW> __host__ __device__ inline size_t tc_smem() {
  constexpr size_t SEG = size_t(NW) * CH;
  // tile, carries, q8 slice + pfend / pbstart slices, published e / b,
  // x-fiber output staging
  return (tc_tile_elems<R, DIM, CH, NW>() + size_t(32 * NW) + 8 * SEG + 2 * NW + 2 * 32 +
          (DIM == 0 ? size_t(NW) * kTcStg : 0)) *
         sizeof(R);
}

#ifndef TC_EPI_B
#define TC_EPI_B 8
#endif
__device__ __forceinline__ void prefetch_l2(const void *p) {
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_count_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;\n" : "=r"(r));
  return r;
}
// generic address of the same shared-memory variable in CTA `rank` of the
// cluster (DSMEM)
template <typename R> __device__ __forceinline__ const R *cluster_peer(const R *p, uint32_t rank) {
  uint64_t out;
  asm volatile("mapa.u64 %0, %1, %2;\n" : "=l"(out) : "l"(p), "r"(rank));
  return reinterpret_cast<const R *>(out);
}

template <typename R, int DIM, int CH, int CL, int NW>
__global__ void __launch_bounds__(32 * NW, NW == 8 ? (sizeof(R) == 4 ? 4 : 2) : 1)
    thomas_cluster_kernel(R *__restrict__ f, ThomasLean<R> t, uint64_t nfib, uint32_t m0,
                          uint32_t m1, Epi epi, const R *base, R *out) {
  pdl_wait();
  constexpr int NF = 32, NT = 32 * NW, NCH = NW * CL;
  constexpr uint32_t SEG = uint32_t(NW) * CH, P0 = SEG + 1;
  extern __shared__ __align__(16) unsigned char tc_raw[];
  R *tile = reinterpret_cast<R *>(tc_raw);
  R *carry = tile + tc_tile_elems<R, DIM, CH, NW>();
  R *sq = carry + NT;             // q8 of the segment's positions
  R *spf = sq + 8 * SEG;          // pfend of the segment's chunks
  R *spb = spf + NW;              // pbstart of the segment's chunks
  R *pub_e = spb + NW;            // published forward end values [NF]
  R *pub_b = pub_e + NF;          // published backward start values [NF]
  R *ostg = pub_b + NF;           // x fibers: per-warp output staging
  const uint32_t m = t.m;
  const uint32_t mp = uint32_t(NCH) * CH;
  const R *gq = t.tab, *gpf = gq + 8 * size_t(mp), *gpb = gpf + NCH, *gmf = gpb + NCH,
          *gmb = gmf + CL;
  const int tid = threadIdx.x, fi = tid % NF, w = tid / NF, lane = tid & 31;
  const uint32_t r = cluster_rank();
  const uint64_t ngroups = (nfib + NF - 1) / NF;
  const uint64_t gstep = cluster_count_x();
  const uint32_t pa0 = r * SEG;
  const uint32_t plen = pa0 >= m ? 0u : (m - pa0 < SEG ? m - pa0 : SEG);
  const uint32_t a = uint32_t(w) * CH; // local chunk start
  const uint32_t len = a >= plen ? 0u : (plen - a < uint32_t(CH) ? plen - a : uint32_t(CH));
  const uint64_t m01 = uint64_t(m0) * m1;
  const uint64_t ps = DIM == 1 ? m0 : m01; // position stride (DIM 1, 2)
  // position-0 address of fiber `fi` of group `gi` (DIM 1, 2; fibers past the
  // end repeat the last)
  auto fiber_addr = [&](uint64_t gi) -> uint64_t {
    const uint64_t F0 = gi * NF;
    const uint64_t F = F0 + min(uint64_t(fi), nfib - 1 - F0);
    return DIM == 1 ? (F % m0) + m01 * (F / m0) : F;
  };
  auto stage = [&](uint64_t gi) {
    const uint64_t F0 = gi * NF;
    const int nf = int(nfib - F0 < uint64_t(NF) ? nfib - F0 : uint64_t(NF));
    if (DIM == 0) {
      for (int row = w; row < nf; row += NW) {
        const R *src = f + (F0 + row) * m + pa0;
        for (uint32_t j = lane; j < plen; j += 32)
          cp_async(tile + size_t(row) * P0 + j, src + j);
      }
    } else {
      const uint64_t fa = fiber_addr(gi);
      for (uint32_t i = w; i < plen; i += NW)
        cp_async(tile + size_t(i) * NF + fi, f + fa + ps * (pa0 + i));
    }
    cp_async_commit();
  };

  uint64_t gi = cluster_id_x();
  tf_copy_in<R, NT>(sq, gq + 8 * size_t(pa0), 8 * SEG, tid); // 8*pa0*sizeof(R): 16-byte multiple
  if (tid < NW) {
    spf[tid] = gpf[r * NW + tid];
    spb[tid] = gpb[r * NW + tid];
  }
  if (gi < ngroups)
    stage(gi);
  const R *qa = sq + 8 * size_t(a);
  for (; gi < ngroups; gi += gstep) {
    const uint64_t F0 = gi * NF;
    const int nf = int(nfib - F0 < uint64_t(NF) ? nfib - F0 : uint64_t(NF));
    cp_async_wait<0>();
    __syncthreads();
    R v[CH];
    {
      const uint32_t ln = (DIM == 0 && fi >= nf) ? 0u : len;
#pragma unroll
      for (int k = 0; k < CH; ++k)
        v[k] = uint32_t(k) < ln ? (DIM == 0 ? tile[size_t(fi) * P0 + a + k]
                                            : tile[size_t(a + k) * NF + fi])
                                : R(0);
    }
    __syncthreads(); // the tile is free: the next group's rows go in now
    if (gi + gstep < ngroups)
      stage(gi + gstep);
    // x fibers: the epilogue's base values pulled into L2 now, read after
    // the solve (y / z fibers: measured slower -- 33 prefetches per thread)
    if (DIM == 0 && epi != Epi::none && fi < nf) {
      const R *bp = base + (F0 + fi) * m + pa0 + a;
#pragma unroll
      for (int k = 0; k < CH; k += 32 / int(sizeof(R)))
        if (uint32_t(k) < len)
          prefetch_l2(bp + k);
    }

    // ---- forward, zero carry-in; publish the segment's end value
    R acc = R(0);
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      acc = fma(qa[8 * k], acc, v[k]);
      v[k] = acc;
    }
    carry[w * NF + fi] = acc;
    __syncthreads();
    if (w == 0) {
      R e = R(0);
#pragma unroll
      for (int k = 0; k < NW; ++k)
        e = fma(spf[k], e, carry[k * NF + fi]);
      pub_e[fi] = e;
    }
    cluster_arrive();
    cluster_wait();
    R c = R(0);
#pragma unroll
    for (int q = 0; q < CL - 1; ++q)
      if (uint32_t(q) < r)
        c = fma(gmf[q], c, cluster_peer(pub_e, uint32_t(q))[fi]);
    for (int k = 0; k < w; ++k)
      c = fma(spf[k], c, carry[k * NF + fi]);

    // ---- forward fix-up + backward, zero carry-in; publish the segment start
    R x = R(0);
#pragma unroll
    for (int k = CH - 1; k >= 0; --k) {
      const R *q = qa + 8 * k;
      const R vj = fma(q[3], c, v[k]);
      x = fma(q[2], x, q[1] * vj);
      v[k] = x;
    }
    __syncthreads(); // every thread has read the forward carries
    carry[w * NF + fi] = x;
    __syncthreads();
    if (w == 0) {
      R b = R(0);
#pragma unroll
      for (int k = NW - 1; k >= 0; --k)
        b = fma(spb[k], b, carry[k * NF + fi]);
      pub_b[fi] = b;
    }
    cluster_arrive();
    cluster_wait();
    R d = R(0);
#pragma unroll
    for (int q = CL - 1; q > 0; --q)
      if (uint32_t(q) > r)
        d = fma(gmb[q], d, cluster_peer(pub_b, uint32_t(q))[fi]);
    for (int k = NW - 1; k > w; --k)
      d = fma(spb[k], d, carry[k * NF + fi]);

    // ---- backward fix-up, epilogue, store (registers -> HBM)
#pragma unroll
    for (int k = 0; k < CH; ++k)
      v[k] = fma(qa[8 * k + 4], d, v[k]);
    if (DIM == 0) {
      // through the warp's staging, 8 positions at a time: a store
      // instruction then covers 4 fibers x 8 consecutive positions (4
      // 8-element runs) instead of 32 scattered elements
      R *stg = ostg + w * kTcStg;
      const int pos = lane & 7, fq = lane >> 3;
#pragma unroll
      for (int k0 = 0; k0 < CH; k0 += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (k0 + j < CH)
            stg[fi * 9 + j] = v[k0 + j];
        __syncwarp();
        if (uint32_t(k0 + pos) < len) {
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int fb = it * 4 + fq;
            if (fb < nf) {
              const uint64_t g = (F0 + fb) * m + pa0 + a + k0 + pos;
              const R z = stg[fb * 9 + pos];
              if (epi == Epi::none)
                f[g] = z;
              else
                out[g] = epi == Epi::add ? base[g] + z : base[g] - z;
            }
          }
        }
        __syncwarp();
      }
    } else if (fi < nf) {
      const uint64_t p0 = fiber_addr(gi) + ps * (pa0 + a), st = ps;
      R *o = (epi == Epi::none ? f : out) + p0;
      if (epi == Epi::none) {
#pragma unroll
        for (int k = 0; k < CH; ++k)
          if (uint32_t(k) < len)
            o[k * st] = v[k];
      } else {
        const R *bp = base + p0;
        constexpr int B = TC_EPI_B; // base loads in flight per batch
#pragma unroll
        for (int k0 = 0; k0 < CH; k0 += B) {
          R bv[B];
#pragma unroll
          for (int k = 0; k < B; ++k)
            if (k0 + k < CH && uint32_t(k0 + k) < len)
              bv[k] = __ldcs(bp + (k0 + k) * st);
#pragma unroll
          for (int k = 0; k < B; ++k)
            if (k0 + k < CH && uint32_t(k0 + k) < len)
              o[(k0 + k) * st] = epi == Epi::add ? bv[k] + v[k0 + k] : bv[k] - v[k0 + k];
        }
      }
    }
  }
  cluster_arrive();
  cluster_wait(); // no CTA leaves while a peer may still read its carries
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
