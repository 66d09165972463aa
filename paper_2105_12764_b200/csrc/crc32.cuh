// crc32.cuh -- CRC-32 (reflected, polynomial 0xEDB88320, init and final xor
// 0xFFFFFFFF: mgr::crc32, /root/reference/proj/src/pipeline.cpp:13-28, the
// same function as zlib's crc32) of device buffers, for the MGRF container's
// per-class records (pipeline.cpp:180-200).
//
// CRC is affine over GF(2): with crc0(X) the register after processing X
// from a zero register, and Z_n the linear map "feed n zero bytes",
//   crc0(A || B) = Z_|B|(crc0(A)) ^ crc0(B),
//   crc(X)       = Z_|X|(0xFFFFFFFF) ^ crc0(X) ^ 0xFFFFFFFF.
// A 32x32 GF(2) matrix applied to a register is kept as four 256-entry byte
// tables (M v = T0[v & 255] ^ T1[v >> 8 & 255] ^ T2[..] ^ T3[v >> 24]).
//
//   crc_blocks_kernel: every warp owns a contiguous segment of 2^seglog blocks
//     of 512 bytes; per block each lane folds its 16 bytes (one coalesced
//     16-byte load per lane, slice-by-4 tables), the 32 lane values combine
//     in 5 butterfly steps (Z_16, Z_32, ..., Z_256), and the block value is
//     accumulated into the segment value with Z_512.
//   crc_combine_kernel (one CTA): thread t folds a run of consecutive
//     segment values with Z_seg, thread 0 folds the 1024 run values with
//     Z_run, the partial last segment and the tail bytes (< 512), then adds
//     the init term.  HBM traffic: the buffer is read once.
#pragma once

#include <cstdint>

namespace mgrg {

__device__ __forceinline__ uint64_t u64min(uint64_t a, uint64_t b) { return a < b ? a : b; }

constexpr int kCrcSegMaxLog = 8; // 512-byte blocks per warp segment: 2^seglog, 8..256
constexpr int kCrcSegMinLog = 3; //   (host-chosen per range: enough segments for every warp)
constexpr int kCrcWarps = 8;       // warps per CTA of the block kernel
constexpr int kCrcRuns = 1024;     // threads of the combine kernel

// Several byte ranges (the class records of one container) in one launch:
// the segments of every range are numbered consecutively (seg0), a warp's
// global segment id picks its range by a short scan.
constexpr int kCrcMaxRanges = 32;
struct CrcRange {
  const uint4 *data; // 16-byte aligned body
  uint64_t nblk;     // 512-byte blocks
  uint64_t seg0;     // first global segment id
  uint32_t *seg;     // segment values
  int seglog;        // 2^seglog blocks per segment
};
struct CrcJobs {
  CrcRange r[kCrcMaxRanges];
  int n;
  uint64_t nseg; // total segments
};
__device__ __forceinline__ int crc_range_of(const CrcJobs &J, uint64_t gsid) {
  int ri = 0;
  while (ri + 1 < J.n && gsid >= J.r[ri + 1].seg0)
    ++ri;
  return ri;
}

// Device tables (uploaded once per process, crc_tables()):
//   slice[4][256]            slice-by-4 CRC tables
//   z16, z32, z64, z128, z256 butterfly shifts; z512 per-block accumulation;
//   zb[k] = Z_{512 * 2^k}, k < 32 (partial last segment, run lengths)
struct CrcTables {
  uint32_t slice[4][256];
  uint32_t z[6][4][256]; // Z_16 .. Z_512
  uint32_t zb[32][4][256];
};


// crc0 of 16 bytes (4 little-endian words), slice-by-4 in shared memory
__device__ __forceinline__ uint32_t crc_fold16(const uint32_t (*s)[256], uint4 w) {
  uint32_t c = 0;
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    c ^= ws[i];
    c = s[3][c & 255u] ^ s[2][(c >> 8) & 255u] ^ s[1][(c >> 16) & 255u] ^ s[0][c >> 24];
  }
  return c;
}

// seg[i] = crc0 of segment i (2^seglog blocks of 512 B; the last one
// may be shorter: nblk total blocks).  Lane a folds the 16 bytes it owns in
// every block and accumulates them Horner-style across the segment's blocks
// (acc = Z_512(acc) ^ piece: its pieces are 512 bytes apart), so the lanes
// never talk inside the loop; one butterfly at the end places lane a's
// stream at its byte offset (Z_{16 * (31 - a)} overall).  Tables in shared
// memory: slice-by-4 for the folds, Z_512 and the butterfly shifts.
__global__ void __launch_bounds__(32 * kCrcWarps)
    crc_blocks_kernel(const __grid_constant__ CrcJobs J, const CrcTables *__restrict__ T) {
  __shared__ uint32_t s[4][256];
  __shared__ uint32_t z[6][4][256];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x)
    s[i >> 8][i & 255] = T->slice[i >> 8][i & 255];
  for (int i = threadIdx.x; i < 6 * 1024; i += blockDim.x)
    (&z[0][0][0])[i] = (&T->z[0][0][0])[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  auto zap = [&](int k, uint32_t v) {
    return z[k][0][v & 255u] ^ z[k][1][(v >> 8) & 255u] ^ z[k][2][(v >> 16) & 255u] ^
           z[k][3][v >> 24];
  };
  // persistent warps: the tables are staged once per CTA
  for (uint64_t gsid = uint64_t(blockIdx.x) * kCrcWarps + (threadIdx.x >> 5); gsid < J.nseg;
       gsid += uint64_t(gridDim.x) * kCrcWarps) {
  const CrcRange &R = J.r[crc_range_of(J, gsid)];
  const uint4 *data = R.data;
  const uint64_t sid = gsid - R.seg0, segb = uint64_t(1) << R.seglog;
  const uint64_t b0 = sid * segb, b1 = u64min(b0 + segb, R.nblk);
  uint32_t acc = 0;
  uint64_t b = b0;
  // four blocks per iteration: the loads and the four independent folds
  // overlap; only the Horner accumulation is a chain
  for (; b + 3 < b1; b += 4) {
    const uint4 w0 = __ldg(data + b * 32 + lane), w1 = __ldg(data + (b + 1) * 32 + lane);
    const uint4 w2 = __ldg(data + (b + 2) * 32 + lane), w3 = __ldg(data + (b + 3) * 32 + lane);
    const uint32_t f0 = crc_fold16(s, w0), f1 = crc_fold16(s, w1);
    const uint32_t f2 = crc_fold16(s, w2), f3 = crc_fold16(s, w3);
    acc = zap(5, acc) ^ f0;
    acc = zap(5, acc) ^ f1;
    acc = zap(5, acc) ^ f2;
    acc = zap(5, acc) ^ f3;
  }
  for (; b < b1; ++b)
    acc = zap(5, acc) ^ crc_fold16(s, __ldg(data + b * 32 + lane));
  // lane a's stream ends 16 * (31 - a) bytes before the segment's end
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const uint32_t r = __shfl_down_sync(0xffffffffu, acc, 1 << k);
    acc = zap(k, acc) ^ r; // Z_{16 * 2^k}(left) ^ right
  }
  if (lane == 0)
    R.seg[sid] = acc;
  }
}

// Same segment values from a kernel whose slice-by-4 lookups never conflict:
// every lane owns a private copy of the four slice tables laid out so that
// lane a's entries all sit in bank a (word (t*256 + e)*32 + a: 128 KiB, one
// CTA of 16 warps per SM).  The shared tables of the previous kernel were
// bound by bank conflicts of 32 random lookups per warp instruction (ncu:
// 26 % DRAM, 27 % issue).  Lane a owns bytes [64a, 64a + 64) of every 2 KiB
// quad of blocks (four 16-byte loads) and accumulates with Z_2048, so one
// conflicted Z lookup set is paid per 64 bytes; the butterfly places the
// lane streams with Z_64 .. Z_1024.  A segment whose block count is not a
// multiple of 4 ends with 1-3 single blocks, folded the old way (16 bytes
// per lane, Z_512 Horner, Z_16 .. Z_256 butterfly) and appended.
constexpr int kCrc2Warps = 16;
__host__ __device__ constexpr size_t crc2_smem() {
  return (4 * 256 * 32 + 8 * 4 * 256) * sizeof(uint32_t);
}
__global__ void __launch_bounds__(32 * kCrc2Warps, 1)
    crc_blocks2_kernel(const __grid_constant__ CrcJobs J, const CrcTables *__restrict__ T) {
  extern __shared__ uint32_t crc2_sm[];
  uint32_t *ls = crc2_sm;                    // [4][256][32] lane-private slice tables
  uint32_t(*z)[4][256] = reinterpret_cast<uint32_t(*)[4][256]>(crc2_sm + 4 * 256 * 32);
  // z[0..5] = Z_16 .. Z_512, z[6] = Z_1024, z[7] = Z_2048
  for (int i = threadIdx.x; i < 4 * 256 * 32; i += blockDim.x)
    ls[i] = (&T->slice[0][0])[i >> 5];
  for (int i = threadIdx.x; i < 6 * 1024; i += blockDim.x)
    (&z[0][0][0])[i] = (&T->z[0][0][0])[i];
  for (int i = threadIdx.x; i < 2 * 1024; i += blockDim.x)
    (&z[6][0][0])[i] = (&T->zb[1][0][0])[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t *lp = ls + lane;
  auto fold_word = [&](uint32_t c) {
    return lp[(3 * 256 + (c & 255u)) << 5] ^ lp[(2 * 256 + ((c >> 8) & 255u)) << 5] ^
           lp[(1 * 256 + ((c >> 16) & 255u)) << 5] ^ lp[(c >> 24) << 5];
  };
  auto fold16 = [&](uint4 w, uint32_t c) {
    c = fold_word(c ^ w.x);
    c = fold_word(c ^ w.y);
    c = fold_word(c ^ w.z);
    return fold_word(c ^ w.w);
  };
  auto zap = [&](int k, uint32_t v) {
    return z[k][0][v & 255u] ^ z[k][1][(v >> 8) & 255u] ^ z[k][2][(v >> 16) & 255u] ^
           z[k][3][v >> 24];
  };
  for (uint64_t gsid = uint64_t(blockIdx.x) * kCrc2Warps + (threadIdx.x >> 5); gsid < J.nseg;
       gsid += uint64_t(gridDim.x) * kCrc2Warps) {
    const CrcRange &R = J.r[crc_range_of(J, gsid)];
    const uint4 *data = R.data;
    const uint64_t sid = gsid - R.seg0, segb = uint64_t(1) << R.seglog;
    const uint64_t b0 = sid * segb, b1 = u64min(b0 + segb, R.nblk);
    const uint64_t nquad = (b1 - b0) / 4;
    const uint4 *dp = data + b0 * 32 + 4 * lane;
    uint32_t acc = 0;
    uint64_t q = 0;
    // two quads per iteration: eight loads in flight, two independent folds
    for (; q + 1 < nquad; q += 2) {
      const uint4 *a = dp + q * 128;
      const uint4 w0 = __ldg(a), w1 = __ldg(a + 1), w2 = __ldg(a + 2), w3 = __ldg(a + 3);
      const uint4 w4 = __ldg(a + 128), w5 = __ldg(a + 129), w6 = __ldg(a + 130),
                  w7 = __ldg(a + 131);
      const uint32_t f0 = fold16(w3, fold16(w2, fold16(w1, fold16(w0, 0u))));
      const uint32_t f1 = fold16(w7, fold16(w6, fold16(w5, fold16(w4, 0u))));
      acc = zap(7, acc) ^ f0;
      acc = zap(7, acc) ^ f1;
    }
    if (q < nquad) {
      const uint4 *a = dp + q * 128;
      acc = zap(7, acc) ^
            fold16(__ldg(a + 3), fold16(__ldg(a + 2), fold16(__ldg(a + 1), fold16(__ldg(a), 0u))));
    }
    // lane a's 64-byte stream ends 64 * (31 - a) bytes before the quads' end
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const uint32_t r = __shfl_down_sync(0xffffffffu, acc, 1 << k);
      acc = zap(2 + k, acc) ^ r; // Z_{64 * 2^k}(left) ^ right
    }
    const int rem = int((b1 - b0) & 3);
    if (rem) { // trailing single blocks: 16 bytes per lane
      uint32_t h = 0;
      for (uint64_t b = b0 + 4 * nquad; b < b1; ++b)
        h = zap(5, h) ^ fold16(__ldg(data + b * 32 + lane), 0u);
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const uint32_t r = __shfl_down_sync(0xffffffffu, h, 1 << k);
        h = zap(k, h) ^ r;
      }
      // append: Z_{512 * rem}(quads) ^ singles
      acc = rem == 1 ? zap(5, acc) : (rem == 2 ? zap(6, acc) : zap(6, zap(5, acc)));
      acc ^= h;
    }
    if (lane == 0)
      R.seg[sid] = acc;
  }
}


// One CTA per range: thread t folds a run of per = 2^p consecutive segment values
// (<= 1024 runs; full segments shift by the staged single table
// Z_{512 * SEG}), the runs meet in a 10-level tree (round 1 folded them
// serially on thread 0: ~50 us per call), then thread 0 adds the head bytes,
// the tail bytes, the init term (zinit = Z_n(0xFFFFFFFF), host-computed) and
// the final xor.
struct CrcFin {
  const uint32_t *seg;
  uint64_t nseg, nblk;
  int seglog;
  const uint8_t *head, *tail;
  uint32_t nhead, ntail, zinit;
  uint32_t *out;
};
struct CrcFins {
  CrcFin f[kCrcMaxRanges];
  int n;
};
constexpr size_t crc_combine_smem() { return (32 + 1) * 4 * 256 * sizeof(uint32_t); }
__global__ void __launch_bounds__(kCrcRuns)
    crc_combine_kernel(const __grid_constant__ CrcFins FS, const CrcTables *__restrict__ T) {
  // one CTA per range
  const CrcFin &FN = FS.f[blockIdx.x];
  const uint32_t *seg = FN.seg;
  const uint64_t nseg = FN.nseg, nblk = FN.nblk;
  const int seglog = FN.seglog;
  const uint8_t *head = FN.head, *tail = FN.tail;
  const uint32_t nhead = FN.nhead, ntail = FN.ntail, zinit = FN.zinit;
  uint32_t *out = FN.out;
  __shared__ uint32_t run[kCrcRuns];
  // every table this kernel touches, staged once (the lookups of the tree
  // and of the byte loops are dependent chains: shared-memory latency)
  extern __shared__ uint32_t cc_sm[];
  uint32_t(*zb)[4][256] = reinterpret_cast<uint32_t(*)[4][256]>(cc_sm); // Z_{512 * 2^k}
  uint32_t(*sl)[256] = reinterpret_cast<uint32_t(*)[256]>(cc_sm + 32 * 1024); // slice-by-4
  for (int i = threadIdx.x; i < 32 * 1024; i += blockDim.x)
    (&zb[0][0][0])[i] = (&T->zb[0][0][0])[i];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x)
    (&sl[0][0])[i] = (&T->slice[0][0])[i];
  int p = 0;
  while ((uint64_t(kCrcRuns) << p) < nseg)
    ++p;
  const uint64_t per = uint64_t(1) << p, segb = uint64_t(1) << seglog;
  __syncthreads();
  auto ap = [](const uint32_t (*z)[256], uint32_t v) {
    return z[0][v & 255u] ^ z[1][(v >> 8) & 255u] ^ z[2][(v >> 16) & 255u] ^ z[3][v >> 24];
  };
  auto zblocks = [&](uint32_t v, uint64_t nb) { // Z_{512 * nb}
    for (int k = 0; nb; ++k, nb >>= 1)
      if (nb & 1)
        v = ap(zb[k], v);
    return v;
  };
  const int t = threadIdx.x;
  const uint64_t s0 = u64min(uint64_t(t) * per, nseg), s1 = u64min(s0 + per, nseg);
  uint32_t v = 0;
  for (uint64_t i = s0; i < s1; ++i) {
    // segment i spans blocks [i*SEG, min((i+1)*SEG, nblk))
    const uint64_t nb = u64min(segb, nblk - i * segb);
    v = (nb == segb ? ap(zb[seglog], v) : zblocks(v, nb)) ^ seg[i];
  }
  run[t] = v;
  __syncthreads();
  // fold the runs pairwise in a tree: at stride w, run t (t % 2w == 0) takes
  // run t + w, whose group spans blocks [(t + w) * per, (t + 2w) * per) ∩ body;
  // full groups shift by one table, the group holding the partial end by
  // binary decomposition
  const uint64_t full = per * segb;
  for (int w = 1, lw = 0; w < kCrcRuns; w <<= 1, ++lw) {
    if ((t & (2 * w - 1)) == 0 && uint64_t(t + w) * per < nseg) {
      const uint64_t g0 = uint64_t(t + w) * full;
      const uint64_t g1 = u64min(uint64_t(t + 2 * w) * full, nblk);
      const uint64_t nb = g1 - g0;
      const int k = seglog + p + lw;
      run[t] = (nb == uint64_t(w) * full && k < 32 ? ap(zb[k], run[t]) : zblocks(run[t], nb)) ^
               run[t + w];
    }
    __syncthreads();
  }
  if (t != 0)
    return;
  // bytes before the 16-byte aligned body, then the body (its crc0 is run[0]:
  // the bytes before it shift by Z_body), then the tail: whole words by
  // slice-by-4, the last bytes one at a time
  uint32_t c = 0;
  for (uint32_t i = 0; i < nhead; ++i) {
    c ^= head[i];
    c = sl[0][c & 255u] ^ (c >> 8);
  }
  c = zblocks(c, nblk) ^ run[0];
  uint32_t i = 0;
  for (; i + 4 <= ntail; i += 4) { // tail starts 16-byte aligned
    c ^= *reinterpret_cast<const uint32_t *>(tail + i);
    c = sl[3][c & 255u] ^ sl[2][(c >> 8) & 255u] ^ sl[1][(c >> 16) & 255u] ^ sl[0][c >> 24];
  }
  for (; i < ntail; ++i) {
    c ^= tail[i];
    c = sl[0][c & 255u] ^ (c >> 8);
  }
  *out = c ^ zinit ^ 0xFFFFFFFFu;
}

} // namespace mgrg
