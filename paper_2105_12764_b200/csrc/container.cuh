// container.cuh -- MGRF container I/O straight from / into the device class
// buffer, with the per-class CRC-32 records computed on the GPU (SURVEY.md
// §8(f) row 1).  Included by mgrg.cu after the plan definition.
//
// On-disk layout (reference include/mgr/pipeline.hpp:27-39, written by
// write_refactored_impl, src/pipeline.cpp:180-206; all little-endian):
//   "MGRF" | u8 version 1 | u8 endianness 0 | u8 dtype (4|8) | u8 ndims
//   | u64 size per dim | f64 coordinates per dim | u64 L
//   | (L+1) x { u64 payload bytes, u32 crc32 } | payloads: class 0 .. class L
// The device class buffer already is the payload sequence (class l at
// N_{l-1}), so writing is: GPU CRCs -> header -> double-buffered D2H chunks
// to the file; reading mirrors read_refactored (pipeline.cpp:233-300): a
// bounded header read, the requested class prefix only, CorruptFile on a CRC
// mismatch (checked on the GPU), MissingClass on a truncated payload.
#pragma once

#include <cstdio>
#include <map>
#include <mutex>

#include "crc32.cuh"

namespace {

// ---- CRC tables (host construction, one device copy per device) ----------
struct GfMat {
  uint32_t col[32]; // image of bit j
};
uint32_t gf_apply(const GfMat &M, uint32_t v) {
  uint32_t r = 0;
  for (int j = 0; j < 32; ++j)
    if ((v >> j) & 1u)
      r ^= M.col[j];
  return r;
}
GfMat gf_compose(const GfMat &A, const GfMat &B) { // A o B
  GfMat C;
  for (int j = 0; j < 32; ++j)
    C.col[j] = gf_apply(A, B.col[j]);
  return C;
}
const uint32_t *crc_table0() {
  static uint32_t t[256];
  static bool init = [] {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k)
        c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      t[i] = c;
    }
    return true;
  }();
  (void)init;
  return t;
}
// Z_{2^k} bytes, k < 64
const std::vector<GfMat> &crc_zpow2() {
  static std::vector<GfMat> z = [] {
    std::vector<GfMat> v(64);
    const uint32_t *t0 = crc_table0();
    for (int j = 0; j < 32; ++j) { // one zero byte
      const uint32_t c = 1u << j;
      v[0].col[j] = t0[c & 255u] ^ (c >> 8);
    }
    for (int k = 1; k < 64; ++k)
      v[k] = gf_compose(v[k - 1], v[k - 1]);
    return v;
  }();
  return z;
}
uint32_t crc_zbytes(uint64_t n, uint32_t v) {
  const auto &z = crc_zpow2();
  for (int k = 0; n; ++k, n >>= 1)
    if (n & 1)
      v = gf_apply(z[k], v);
  return v;
}
void gf_tables(const GfMat &M, uint32_t t[4][256]) {
  for (int k = 0; k < 4; ++k)
    for (uint32_t i = 0; i < 256; ++i)
      t[k][i] = gf_apply(M, i << (8 * k));
}

mgrg_status crc_tables_device(int device, const mgrg::CrcTables **out) {
  static std::mutex mu;
  static std::map<int, mgrg::CrcTables *> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(device);
  if (it != cache.end()) {
    *out = it->second;
    return MGRG_OK;
  }
  std::unique_ptr<mgrg::CrcTables> h(new mgrg::CrcTables());
  const uint32_t *t0 = crc_table0();
  for (int i = 0; i < 256; ++i)
    h->slice[0][i] = t0[i];
  for (int k = 1; k < 4; ++k)
    for (int i = 0; i < 256; ++i)
      h->slice[k][i] = (h->slice[k - 1][i] >> 8) ^ t0[h->slice[k - 1][i] & 255u];
  const auto &z = crc_zpow2();
  for (int k = 0; k < 6; ++k) // Z_16 .. Z_512
    gf_tables(z[4 + k], h->z[k]);
  for (int k = 0; k < 32; ++k) // Z_{512 * 2^k}
    gf_tables(z[9 + k], h->zb[k]);
  mgrg::CrcTables *d = nullptr;
  CUDA_TRY(cudaMalloc(&d, sizeof(mgrg::CrcTables)));
  CUDA_TRY(cudaMemcpy(d, h.get(), sizeof(mgrg::CrcTables), cudaMemcpyHostToDevice));
  cache[device] = d;
  *out = d;
  return MGRG_OK;
}

// lane-private-table segment kernel (crc_blocks2_kernel); MGRG_CRC_V2=0
// selects the shared-table kernel (A/B)
int g_crc_v2 = knob("MGRG_CRC_V2", 1);

// CRC-32 of `count` device byte ranges (ptr[i], len[i]) -> host crc[i]:
// per batch of up to kCrcMaxRanges ranges, one segment launch per kernel
// family (lane-private tables for ranges of >= 2^16 blocks: their ~10 us
// table staging pays off; shared tables below) and one combine launch with a
// CTA per range.
mgrg_status crc32_ranges(int device, const uint8_t *const *ptr, const uint64_t *len,
                         int count, uint32_t *crc, cudaStream_t s) {
  const mgrg::CrcTables *T = nullptr;
  if (mgrg_status st = crc_tables_device(device, &T))
    return st;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  // (per call: the attributes belong to the current device's context)
  if (cudaFuncSetAttribute(mgrg::crc_blocks2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(mgrg::crc2_smem())) != cudaSuccess ||
      cudaFuncSetAttribute(mgrg::crc_combine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(mgrg::crc_combine_smem())) != cudaSuccess)
    return fail(MGRG_CUDA_ERROR, "crc kernels: shared memory attribute");
  struct Plan1 {
    uint64_t head, nblk, tail, nseg;
    int seglog;
    bool v2;
  };
  std::vector<Plan1> pl(count);
  uint64_t words = 0;
  for (int i = 0; i < count; ++i) {
    const uint8_t *d = ptr[i];
    const uint64_t n = len[i];
    Plan1 &q = pl[i];
    q.head = std::min<uint64_t>(n, (16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15);
    q.nblk = (n - q.head) / 512;
    q.tail = n - q.head - q.nblk * 512;
    q.v2 = g_crc_v2 && q.nblk >= (uint64_t(1) << 16);
    // segment length: the largest power of two (8..256 blocks) that still
    // gives every warp of a full wave a segment (small ranges: short serial
    // Horner chains; large ones: few segment values to combine)
    const uint64_t warps = uint64_t(sms) * (q.v2 ? mgrg::kCrc2Warps : 6 * mgrg::kCrcWarps);
    q.seglog = mgrg::kCrcSegMaxLog;
    while (q.seglog > mgrg::kCrcSegMinLog && (q.nblk >> q.seglog) < warps)
      --q.seglog;
    q.nseg = (q.nblk + (uint64_t(1) << q.seglog) - 1) >> q.seglog;
    words += q.nseg + 1;
  }
  uint32_t *scratch = nullptr;
  CUDA_TRY(cudaMallocAsync(&scratch, (words + count) * sizeof(uint32_t), s));
  uint32_t *d_out = scratch + words;
  mgrg_status st = MGRG_OK;
  uint64_t woff = 0;
  for (int b0 = 0; b0 < count && !st; b0 += mgrg::kCrcMaxRanges) {
    const int b1 = std::min(count, b0 + mgrg::kCrcMaxRanges);
    mgrg::CrcJobs J1{}, J2{};
    mgrg::CrcFins FS{};
    for (int i = b0; i < b1; ++i) {
      const Plan1 &q = pl[i];
      uint32_t *seg = scratch + woff;
      woff += q.nseg + 1;
      if (q.nblk) {
        mgrg::CrcJobs &J = q.v2 ? J2 : J1;
        J.r[J.n] = {reinterpret_cast<const uint4 *>(ptr[i] + q.head), q.nblk, J.nseg, seg,
                    q.seglog};
        J.nseg += q.nseg;
        ++J.n;
      }
      FS.f[FS.n++] = {seg,
                      q.nseg,
                      q.nblk,
                      q.seglog,
                      ptr[i],
                      ptr[i] + q.head + q.nblk * 512,
                      uint32_t(q.head),
                      uint32_t(q.tail),
                      crc_zbytes(len[i], 0xFFFFFFFFu),
                      d_out + i};
    }
    if (J2.n)
      mgrg::crc_blocks2_kernel<<<unsigned(std::min<uint64_t>(
                                     (J2.nseg + mgrg::kCrc2Warps - 1) / mgrg::kCrc2Warps,
                                     uint64_t(sms))),
                                 32 * mgrg::kCrc2Warps, mgrg::crc2_smem(), s>>>(J2, T);
    if (J1.n)
      mgrg::crc_blocks_kernel<<<unsigned(std::min<uint64_t>(
                                    (J1.nseg + mgrg::kCrcWarps - 1) / mgrg::kCrcWarps,
                                    uint64_t(sms) * 6)),
                                32 * mgrg::kCrcWarps, 0, s>>>(J1, T);
    mgrg::crc_combine_kernel<<<unsigned(FS.n), mgrg::kCrcRuns, mgrg::crc_combine_smem(), s>>>(
        FS, T);
    if (cudaGetLastError() != cudaSuccess)
      st = fail(MGRG_CUDA_ERROR, "crc kernels: launch failed");
  }
  if (!st) {
    cudaError_t e = cudaMemcpyAsync(crc, d_out, count * sizeof(uint32_t),
                                    cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
      e = cudaStreamSynchronize(s);
    if (e != cudaSuccess)
      st = fail(MGRG_CUDA_ERROR, cudaGetErrorString(e));
  }
  cudaFreeAsync(scratch, s);
  return st;
}

// ---- little-endian header bytes -------------------------------------------
struct LeWriter {
  std::vector<uint8_t> b;
  void u8(uint8_t v) { b.push_back(v); }
  void u32(uint32_t v) {
    for (int i = 0; i < 4; ++i)
      b.push_back(uint8_t(v >> (8 * i)));
  }
  void u64(uint64_t v) {
    for (int i = 0; i < 8; ++i)
      b.push_back(uint8_t(v >> (8 * i)));
  }
  void f64(double v) {
    uint64_t bits;
    std::memcpy(&bits, &v, 8);
    u64(bits);
  }
};
struct LeReader {
  const uint8_t *p;
  size_t n, at = 0;
  bool ok = true;
  const uint8_t *take(size_t k) {
    if (at + k > n) {
      ok = false;
      return nullptr;
    }
    const uint8_t *r = p + at;
    at += k;
    return r;
  }
  uint64_t uint(int bytes) {
    const uint8_t *s = take(bytes);
    uint64_t v = 0;
    if (s)
      for (int i = 0; i < bytes; ++i)
        v |= uint64_t(s[i]) << (8 * i);
    return v;
  }
  double f64() {
    const uint64_t b = uint(8);
    double v;
    std::memcpy(&v, &b, 8);
    return v;
  }
};

uint64_t class_count(const mgrg_plan *p, int l) {
  return l == 0 ? p->nodes[0] : p->nodes[l] - p->nodes[l - 1];
}

struct FileCloser {
  void operator()(FILE *f) const {
    if (f)
      std::fclose(f);
  }
};

} // namespace

extern "C" {

mgrg_status mgrg_crc32(const void *d_bytes, uint64_t nbytes, uint32_t *crc, void *stream) {
  g_last_error.clear();
  if ((!d_bytes && nbytes) || !crc)
    return fail(MGRG_INVALID_ARGUMENT, "null argument");
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  const uint8_t *p = static_cast<const uint8_t *>(d_bytes);
  return crc32_ranges(dev, &p, &nbytes, 1, crc, static_cast<cudaStream_t>(stream));
}

mgrg_status mgrg_class_crc32(mgrg_plan *p, const void *d_classes, int32_t upto,
                             uint32_t *crcs, void *stream) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (!d_classes || !crcs)
    return fail(MGRG_INVALID_ARGUMENT, "null argument");
  if (upto < 0 || upto > p->H.L)
    return fail(MGRG_INVALID_LEVEL, "class index out of range");
  DeviceGuard guard(p->device);
  std::vector<const uint8_t *> ptr(upto + 1);
  std::vector<uint64_t> len(upto + 1);
  const uint8_t *base = static_cast<const uint8_t *>(d_classes);
  for (int l = 0; l <= upto; ++l) {
    ptr[l] = base + (l == 0 ? 0 : p->nodes[l - 1]) * p->esize;
    len[l] = class_count(p, l) * p->esize;
  }
  return crc32_ranges(p->device, ptr.data(), len.data(), upto + 1, crcs,
                      static_cast<cudaStream_t>(stream));
}

mgrg_status mgrg_write_refactored(mgrg_plan *p, const void *d_classes, const char *path,
                                  uint64_t *bytes_written) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (!d_classes || !path)
    return fail(MGRG_INVALID_ARGUMENT, "null argument");
  DeviceGuard guard(p->device);
  if (mgrg_status st = ensure_stage(p))
    return st;
  const int L = p->H.L;
  std::vector<uint32_t> crc(L + 1);
  if (mgrg_status st = mgrg_class_crc32(p, d_classes, L, crc.data(), p->own_stream))
    return st;
  LeWriter w; // write_header, pipeline.cpp:127-143
  for (char c : {'M', 'G', 'R', 'F'})
    w.u8(uint8_t(c));
  w.u8(1);
  w.u8(0);
  w.u8(uint8_t(p->esize));
  w.u8(uint8_t(p->H.nd));
  for (int d = 0; d < p->H.nd; ++d)
    w.u64(p->H.shape[d]);
  for (int d = 0; d < p->H.nd; ++d)
    for (double c : p->H.coords[d])
      w.f64(c);
  w.u64(uint64_t(L));
  for (int l = 0; l <= L; ++l) {
    w.u64(class_count(p, l) * p->esize);
    w.u32(crc[l]);
  }
  std::unique_ptr<FILE, FileCloser> f(std::fopen(path, "wb"));
  if (!f)
    return fail(MGRG_IO_ERROR, std::string("cannot open for writing: ") + path);
  if (std::fwrite(w.b.data(), 1, w.b.size(), f.get()) != w.b.size())
    return fail(MGRG_IO_ERROR, std::string("write failed: ") + path);
  // payloads: double-buffered D2H through pinned chunks, file writes of one
  // chunk overlapping the copy of the next
  const uint64_t total = p->nodes[L] * p->esize;
  const uint64_t chunk = 64ull << 20;
  void *pin[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  mgrg_status st = MGRG_OK;
  for (int i = 0; i < 2 && !st; ++i) {
    if (cudaMallocHost(&pin[i], chunk) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) != cudaSuccess)
      st = fail(MGRG_OUT_OF_MEMORY, "pinned staging for the container write");
  }
  const uint8_t *src = static_cast<const uint8_t *>(d_classes);
  auto issue = [&](uint64_t off, int b) -> bool {
    const uint64_t n = std::min(chunk, total - off);
    return cudaMemcpyAsync(pin[b], src + off, n, cudaMemcpyDeviceToHost, p->own_stream) ==
               cudaSuccess &&
           cudaEventRecord(ev[b], p->own_stream) == cudaSuccess;
  };
  if (!st && total && !issue(0, 0))
    st = fail(MGRG_CUDA_ERROR, "container D2H");
  for (uint64_t off = 0, i = 0; !st && off < total; off += chunk, ++i) {
    const int b = int(i & 1);
    if (off + chunk < total && !issue(off + chunk, b ^ 1)) {
      st = fail(MGRG_CUDA_ERROR, "container D2H");
      break;
    }
    if (cudaEventSynchronize(ev[b]) != cudaSuccess) {
      st = fail(MGRG_CUDA_ERROR, "container D2H");
      break;
    }
    const uint64_t n = std::min(chunk, total - off);
    if (std::fwrite(pin[b], 1, n, f.get()) != n)
      st = fail(MGRG_IO_ERROR, std::string("write failed: ") + path);
  }
  cudaStreamSynchronize(p->own_stream);
  for (int i = 0; i < 2; ++i) {
    if (pin[i])
      cudaFreeHost(pin[i]);
    if (ev[i])
      cudaEventDestroy(ev[i]);
  }
  if (st)
    return st;
  if (std::fflush(f.get()) != 0)
    return fail(MGRG_IO_ERROR, std::string("write failed: ") + path);
  if (bytes_written)
    *bytes_written = w.b.size() + total;
  return MGRG_OK;
}

mgrg_status mgrg_read_refactored(mgrg_plan *p, const char *path, int32_t classes,
                                 void *d_classes, int32_t *classes_loaded,
                                 uint64_t *bytes_consumed) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (!d_classes || !path)
    return fail(MGRG_INVALID_ARGUMENT, "null argument");
  DeviceGuard guard(p->device);
  if (mgrg_status st = ensure_stage(p))
    return st;
  std::unique_ptr<FILE, FileCloser> f(std::fopen(path, "rb"));
  if (!f)
    return fail(MGRG_IO_ERROR, std::string("cannot open: ") + path);
  // read_refactored_header (pipeline.cpp:220-231): one bounded read
  std::vector<uint8_t> hb(1 << 20);
  hb.resize(std::fread(hb.data(), 1, hb.size(), f.get()));
  LeReader r{hb.data(), hb.size()};
  const uint8_t *mg = r.take(4);
  if (!mg)
    return fail(MGRG_CORRUPT_FILE, "unexpected end of data");
  if (std::memcmp(mg, "MGRF", 4) != 0)
    return fail(MGRG_CORRUPT_FILE, "bad magic");
  const uint64_t ver = r.uint(1), endian = r.uint(1), dt = r.uint(1), nd = r.uint(1);
  if (!r.ok)
    return fail(MGRG_CORRUPT_FILE, "unexpected end of data");
  if (ver != 1)
    return fail(MGRG_CORRUPT_FILE, "unsupported version " + std::to_string(ver));
  if (endian != 0)
    return fail(MGRG_CORRUPT_FILE, "unsupported endianness");
  if (dt != 4 && dt != 8)
    return fail(MGRG_CORRUPT_FILE, "unsupported dtype " + std::to_string(dt));
  if (nd < 1 || nd > 4)
    return fail(MGRG_CORRUPT_FILE, "bad dimension count");
  std::vector<uint64_t> shape(nd);
  for (auto &e : shape) {
    e = r.uint(8);
    if (r.ok && e < 2)
      return fail(MGRG_CORRUPT_FILE, "bad dimension size");
  }
  bool coords_match = true;
  for (uint64_t d = 0; d < nd && r.ok; ++d)
    for (uint64_t i = 0; i < shape[d] && r.ok; ++i) {
      const double c = r.f64();
      coords_match = coords_match && int(d) < p->H.nd && i < p->H.coords[d].size() &&
                     std::memcmp(&c, &p->H.coords[d][i], 8) == 0;
    }
  const uint64_t levels = r.uint(8);
  if (!r.ok)
    return fail(MGRG_CORRUPT_FILE, "unexpected end of data");
  if (levels > 64)
    return fail(MGRG_CORRUPT_FILE, "implausible level count");
  std::vector<uint64_t> rb(levels + 1);
  std::vector<uint32_t> rc(levels + 1);
  for (uint64_t l = 0; l <= levels; ++l) {
    rb[l] = r.uint(8);
    rc[l] = uint32_t(r.uint(4));
  }
  if (!r.ok)
    return fail(MGRG_CORRUPT_FILE, "unexpected end of data");
  // the container must be this plan's hierarchy (device buffers have no
  // self-describing type, unlike RefactoredData)
  bool same = int(dt) == p->esize && int(nd) == p->H.nd && int(levels) == p->H.L &&
              coords_match;
  for (uint64_t d = 0; same && d < nd; ++d)
    same = shape[d] == p->H.shape[d];
  for (uint64_t l = 0; same && l <= levels; ++l)
    same = rb[l] == class_count(p, int(l)) * p->esize;
  if (!same)
    return fail(MGRG_INVALID_ARGUMENT,
                "container geometry / dtype / levels do not match the plan");
  const int L = p->H.L;
  const int want = classes < 0 ? L : classes;
  if (want > L)
    return fail(MGRG_MISSING_CLASS, "requested class " + std::to_string(want) +
                                        " of a container with " + std::to_string(L + 1) +
                                        " classes");
  const uint64_t header = r.at;
  if (std::fseek(f.get(), long(header), SEEK_SET) != 0)
    return fail(MGRG_IO_ERROR, std::string("seek failed: ") + path);
  // payload prefix: classes 0..want, double-buffered H2D through pinned chunks
  uint64_t need = 0;
  for (int l = 0; l <= want; ++l)
    need += rb[l];
  const uint64_t chunk = 64ull << 20;
  void *pin[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  mgrg_status st = MGRG_OK;
  for (int i = 0; i < 2 && !st; ++i)
    if (cudaMallocHost(&pin[i], chunk) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) != cudaSuccess)
      st = fail(MGRG_OUT_OF_MEMORY, "pinned staging for the container read");
  uint8_t *dst = static_cast<uint8_t *>(d_classes);
  uint64_t got = 0;
  for (uint64_t i = 0; !st && got < need; ++i) {
    const int b = int(i & 1);
    if (i >= 2 && cudaEventSynchronize(ev[b]) != cudaSuccess) { // buffer b free again
      st = fail(MGRG_CUDA_ERROR, "container H2D");
      break;
    }
    const uint64_t want_n = std::min(chunk, need - got);
    const uint64_t n = std::fread(pin[b], 1, want_n, f.get());
    if (n && (cudaMemcpyAsync(dst + got, pin[b], n, cudaMemcpyHostToDevice, p->own_stream) !=
                  cudaSuccess ||
              cudaEventRecord(ev[b], p->own_stream) != cudaSuccess))
      st = fail(MGRG_CUDA_ERROR, "container H2D");
    got += n;
    if (n < want_n)
      break; // truncated
  }
  cudaStreamSynchronize(p->own_stream);
  for (int i = 0; i < 2; ++i) {
    if (pin[i])
      cudaFreeHost(pin[i]);
    if (ev[i])
      cudaEventDestroy(ev[i]);
  }
  if (st)
    return st;
  // classes fully present, in order; the first truncated one (if any)
  int complete = -1;
  for (uint64_t off = 0; complete < want && off + rb[complete + 1] <= got;)
    off += rb[++complete];
  // CRCs of the complete classes (GPU), first mismatch wins as in the
  // reference's sequential read (pipeline.cpp:271-276)
  if (complete >= 0) {
    std::vector<uint32_t> crc(complete + 1);
    if (mgrg_status s2 = mgrg_class_crc32(p, d_classes, complete, crc.data(), p->own_stream))
      return s2;
    for (int l = 0; l <= complete; ++l)
      if (crc[l] != rc[l])
        return fail(MGRG_CORRUPT_FILE, "crc mismatch in class " + std::to_string(l));
  }
  if (complete < want)
    return fail(MGRG_MISSING_CLASS,
                "class " + std::to_string(complete + 1) + " payload is truncated");
  if (classes_loaded)
    *classes_loaded = want;
  if (bytes_consumed)
    *bytes_consumed = header + need;
  return MGRG_OK;
}

} // extern "C"
