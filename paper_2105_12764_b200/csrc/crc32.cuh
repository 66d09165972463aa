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
//   crc_blocks_kernel: every warp owns a contiguous segment of SEGB blocks
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

constexpr int kCrcSegBlocks = 256; // 512-byte blocks per warp segment (128 KiB)
constexpr int kCrcSegLog = 8;      // log2(kCrcSegBlocks)
constexpr int kCrcWarps = 8;       // warps per CTA of the block kernel
constexpr int kCrcRuns = 1024;     // threads of the combine kernel

// Device tables (uploaded once per process, crc_tables()):
//   slice[4][256]            slice-by-4 CRC tables
//   z16, z32, z64, z128, z256 butterfly shifts; z512 per-block accumulation;
//   zb[k] = Z_{512 * 2^k}, k < 32 (partial last segment, run lengths)
struct CrcTables {
  uint32_t slice[4][256];
  uint32_t z[6][4][256]; // Z_16 .. Z_512
  uint32_t zb[32][4][256];
};

__device__ __forceinline__ uint32_t crc_apply(const uint32_t (*t)[256], uint32_t v) {
  return __ldg(&t[0][v & 255u]) ^ __ldg(&t[1][(v >> 8) & 255u]) ^
         __ldg(&t[2][(v >> 16) & 255u]) ^ __ldg(&t[3][v >> 24]);
}

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

// seg[i] = crc0 of segment i (kCrcSegBlocks blocks of 512 B; the last one
// may be shorter: nblk total blocks).  Lane a folds the 16 bytes it owns in
// every block and accumulates them Horner-style across the segment's blocks
// (acc = Z_512(acc) ^ piece: its pieces are 512 bytes apart), so the lanes
// never talk inside the loop; one butterfly at the end places lane a's
// stream at its byte offset (Z_{16 * (31 - a)} overall).  Tables in shared
// memory: slice-by-4 for the folds, Z_512 and the butterfly shifts.
__global__ void __launch_bounds__(32 * kCrcWarps)
    crc_blocks_kernel(const uint4 *__restrict__ data, uint64_t nblk,
                      const CrcTables *__restrict__ T, uint32_t *__restrict__ seg) {
  __shared__ uint32_t s[4][256];
  __shared__ uint32_t z[6][4][256];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x)
    s[i >> 8][i & 255] = T->slice[i >> 8][i & 255];
  for (int i = threadIdx.x; i < 6 * 1024; i += blockDim.x)
    (&z[0][0][0])[i] = (&T->z[0][0][0])[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t nseg = (nblk + kCrcSegBlocks - 1) / kCrcSegBlocks;
  auto zap = [&](int k, uint32_t v) {
    return z[k][0][v & 255u] ^ z[k][1][(v >> 8) & 255u] ^ z[k][2][(v >> 16) & 255u] ^
           z[k][3][v >> 24];
  };
  // persistent warps: the tables are staged once per CTA
  for (uint64_t sid = uint64_t(blockIdx.x) * kCrcWarps + (threadIdx.x >> 5); sid < nseg;
       sid += uint64_t(gridDim.x) * kCrcWarps) {
  const uint64_t b0 = sid * kCrcSegBlocks, b1 = u64min(b0 + kCrcSegBlocks, nblk);
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
    seg[sid] = acc;
  }
}

// Apply Z_{512 * nb} (nb blocks) by binary decomposition.
__device__ __forceinline__ uint32_t crc_zblocks(const CrcTables *T, uint32_t v, uint64_t nb) {
  for (int k = 0; nb; ++k, nb >>= 1)
    if (nb & 1)
      v = crc_apply(T->zb[k], v);
  return v;
}

// One CTA: fold the head bytes, the segment values in order, then the tail
// bytes, then the init term (zinit = Z_n(0xFFFFFFFF), host-computed) and the
// final xor.  Runs of per = 2^p consecutive segments (one per thread, <= 1024
// runs): full segments fold with Z_{512 * SEG} and full runs with
// Z_{512 * SEG * 2^p} -- both single tables (zb[log SEG], zb[log SEG + p]) staged in
// shared memory -- so thread 0's pass over the runs is short.
__global__ void __launch_bounds__(kCrcRuns)
    crc_combine_kernel(const uint32_t *__restrict__ seg, uint64_t nseg, uint64_t nblk,
                       const uint8_t *__restrict__ head, uint32_t nhead,
                       const uint8_t *__restrict__ tail, uint32_t ntail, uint32_t zinit,
                       const CrcTables *__restrict__ T, uint32_t *__restrict__ out) {
  __shared__ uint32_t run[kCrcRuns];
  __shared__ uint32_t zs[4][256], zr[4][256];
  int p = 0;
  while ((uint64_t(kCrcRuns) << p) < nseg)
    ++p;
  const uint64_t per = uint64_t(1) << p;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    zs[i >> 8][i & 255] = T->zb[kCrcSegLog][i >> 8][i & 255];
    zr[i >> 8][i & 255] = T->zb[kCrcSegLog + p][i >> 8][i & 255];
  }
  __syncthreads();
  auto ap = [](const uint32_t (*z)[256], uint32_t v) {
    return z[0][v & 255u] ^ z[1][(v >> 8) & 255u] ^ z[2][(v >> 16) & 255u] ^ z[3][v >> 24];
  };
  const int t = threadIdx.x;
  const uint64_t s0 = u64min(uint64_t(t) * per, nseg), s1 = u64min(s0 + per, nseg);
  uint32_t v = 0;
  for (uint64_t i = s0; i < s1; ++i) {
    // segment i spans blocks [i*SEG, min((i+1)*SEG, nblk))
    const uint64_t nb = u64min(kCrcSegBlocks, nblk - i * kCrcSegBlocks);
    v = (nb == kCrcSegBlocks ? ap(zs, v) : crc_zblocks(T, v, nb)) ^ seg[i];
  }
  run[t] = v;
  __syncthreads();
  if (t != 0)
    return;
  // bytes before the 16-byte aligned body, then the body's runs (folding a
  // run applies Z_run to everything before it), then the tail
  uint32_t c = 0;
  for (uint32_t i = 0; i < nhead; ++i) {
    c ^= head[i];
    c = T->slice[0][c & 255u] ^ (c >> 8);
  }
  const uint64_t full = per * kCrcSegBlocks;
  for (int r = 0; r < kCrcRuns; ++r) {
    const uint64_t a = u64min(uint64_t(r) * per, nseg), b = u64min(a + per, nseg);
    if (b <= a)
      break;
    const uint64_t nb = u64min(b * kCrcSegBlocks, nblk) - a * kCrcSegBlocks;
    c = (nb == full ? ap(zr, c) : crc_zblocks(T, c, nb)) ^ run[r];
  }
  for (uint32_t i = 0; i < ntail; ++i) {
    c ^= tail[i];
    c = T->slice[0][c & 255u] ^ (c >> 8);
  }
  *out = c ^ zinit ^ 0xFFFFFFFFu;
}

} // namespace mgrg
