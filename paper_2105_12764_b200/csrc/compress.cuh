// compress.cuh -- mgr::compress / mgr::decompress (
// reference include/mgr/pipeline.hpp:149-198, src/pipeline.cpp:381-547) with
// the device doing the refactoring, the quantizer's error-bound search
// (quantize, dequantize, full recompose, max |error| -- every attempt), and
// the zigzag-varint coding; the lossless codec (store / zlib) stays on the
// host as in the paper's Showcase 2.  Included by mgrg.cu.
//
// Container "MGRC" (build_compressed_container, pipeline.cpp:444-474):
//   "MGRC" | u8 1 | u8 codec | u8 dtype | u8 ndims | u64 shape | f64 coords
//   | u64 L | f64 eb | f64 bin | f64 measured
//   | per class: u64 count, u64 raw bytes, u64 encoded bytes, encoded bytes
// With the exact arithmetic policy the quantized classes, the bin sequence
// and therefore the bytes equal the reference's (same zlib).
#pragma once

#include <cub/cub.cuh>
#include <zlib.h>

#include "quantize.cuh"

namespace {

constexpr unsigned kQBlocks = 148 * 8, kQThreads = 256;

mgrg_status codec_encode(int codec, const std::vector<uint8_t> &raw, std::vector<uint8_t> &enc) {
  if (codec == 0) { // StoreCodec (pipeline.cpp:305-320)
    enc = raw;
    return MGRG_OK;
  }
  uLongf bound = compressBound(uLong(raw.size())); // ZlibCodec (:322-346)
  enc.resize(bound);
  if (compress2(enc.data(), &bound, raw.data(), uLong(raw.size()), Z_DEFAULT_COMPRESSION) !=
      Z_OK)
    return fail(MGRG_IO_ERROR, "zlib compression failed");
  enc.resize(bound);
  return MGRG_OK;
}
mgrg_status codec_decode(int codec, const uint8_t *enc, uint64_t n, uint64_t raw_size,
                         std::vector<uint8_t> &raw) {
  if (codec == 0) {
    if (n != raw_size)
      return fail(MGRG_CORRUPT_FILE, "stored block size mismatch");
    raw.assign(enc, enc + n);
    return MGRG_OK;
  }
  raw.resize(raw_size);
  uLongf len = uLongf(raw_size);
  if (uncompress(raw.data(), &len, enc, uLong(n)) != Z_OK || len != raw_size)
    return fail(MGRG_CORRUPT_FILE, "zlib decompression failed");
  return MGRG_OK;
}

template <typename R>
mgrg_status compress_impl(mgrg_plan *p, const R *d_values, double eb, int codec,
                          std::vector<uint8_t> &out, double *bin_out, double *measured_out) {
  const int L = p->H.L;
  const uint64_t N = p->nodes[L];
  cudaStream_t s = p->own_stream;
  R *cls = nullptr, *deq = nullptr, *rec = nullptr;
  int64_t *q = nullptr;
  unsigned long long *dmax = nullptr;
  CUDA_TRY(cudaMallocAsync(&cls, N * sizeof(R), s));
  CUDA_TRY(cudaMallocAsync(&deq, N * sizeof(R), s));
  CUDA_TRY(cudaMallocAsync(&rec, N * sizeof(R), s));
  CUDA_TRY(cudaMallocAsync(&q, N * sizeof(int64_t), s));
  CUDA_TRY(cudaMallocAsync(&dmax, sizeof(unsigned long long), s));
  struct Free {
    cudaStream_t s;
    std::vector<void *> v;
    ~Free() {
      for (void *x : v)
        cudaFreeAsync(x, s);
      cudaStreamSynchronize(s);
    }
  } guard{s, {cls, deq, rec, q, dmax}};
  if (mgrg_status st = run_decompose<R>(p, d_values, cls, s))
    return st;
  // the error-bound search, pipeline.hpp:161-180
  double bin = 2.0 * eb / double(L + 1), measured = 0;
  for (int attempt = 0;; ++attempt) {
    quantize_kernel<R><<<kQBlocks, kQThreads, 0, s>>>(cls, N, bin, q, deq);
    if (mgrg_status st = run_recompose<R>(p, deq, L, rec, s))
      return st;
    CUDA_TRY(cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), s));
    maxabs_kernel<R><<<kQBlocks, kQThreads, 0, s>>>(rec, d_values, N, dmax);
    unsigned long long bits = 0;
    CUDA_TRY(cudaMemcpyAsync(&bits, dmax, sizeof(bits), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    std::memcpy(&measured, &bits, 8);
    if (measured <= eb)
      break;
    if (attempt >= 24)
      return fail(MGRG_INVALID_BOUND, "quantizer failed to reach the requested bound");
    bin *= 0.5;
  }
  // header (build_compressed_container)
  LeWriter w;
  for (char c : {'M', 'G', 'R', 'C'})
    w.u8(uint8_t(c));
  w.u8(1);
  w.u8(uint8_t(codec));
  w.u8(uint8_t(sizeof(R)));
  w.u8(uint8_t(p->H.nd));
  for (int d = 0; d < p->H.nd; ++d)
    w.u64(p->H.shape[d]);
  for (int d = 0; d < p->H.nd; ++d)
    for (double c : p->H.coords[d])
      w.f64(c);
  w.u64(uint64_t(L));
  w.f64(eb);
  w.f64(bin);
  w.f64(measured);
  // per class: zigzag-varint on the device, codec on the host
  uint64_t *len = nullptr;
  uint8_t *raw = nullptr;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, len, len, N + 1, s));
  CUDA_TRY(cudaMallocAsync(&len, (N + 1) * sizeof(uint64_t), s));
  CUDA_TRY(cudaMallocAsync(&raw, N * 10, s));
  CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, s));
  guard.v.push_back(len);
  guard.v.push_back(raw);
  guard.v.push_back(tmp);
  std::vector<uint8_t> hraw, enc;
  for (int l = 0; l <= L; ++l) {
    const uint64_t off = l == 0 ? 0 : p->nodes[l - 1], n = class_count(p, l);
    zz_len_kernel<<<kQBlocks, kQThreads, 0, s>>>(q + off, n, len);
    CUDA_TRY(cudaMemsetAsync(len + n, 0, sizeof(uint64_t), s));
    size_t tb = tmp_bytes;
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, len, len, n + 1, s));
    zz_write_kernel<<<kQBlocks, kQThreads, 0, s>>>(q + off, n, len, raw);
    uint64_t nbytes = 0;
    CUDA_TRY(cudaMemcpyAsync(&nbytes, len + n, sizeof(nbytes), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    hraw.resize(nbytes);
    CUDA_TRY(cudaMemcpyAsync(hraw.data(), raw, nbytes, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (mgrg_status st = codec_encode(codec, hraw, enc))
      return st;
    w.u64(n);
    w.u64(nbytes);
    w.u64(enc.size());
    w.b.insert(w.b.end(), enc.begin(), enc.end());
  }
  out.swap(w.b);
  *bin_out = bin;
  *measured_out = measured;
  return MGRG_OK;
}

template <typename R>
mgrg_status decompress_impl(mgrg_plan *p, const uint8_t *bytes, uint64_t size, R *d_values,
                            double *eb, double *bin_out, double *measured, int32_t *codec_out) {
  // parse_compressed_container (pipeline.cpp:476-515)
  LeReader r{bytes, size_t(size)};
  auto eod = [] { return fail(MGRG_CORRUPT_FILE, "unexpected end of data"); };
  const uint8_t *mg = r.take(4);
  if (!mg)
    return eod();
  if (std::memcmp(mg, "MGRC", 4) != 0)
    return fail(MGRG_CORRUPT_FILE, "bad magic");
  const uint64_t ver = r.uint(1), codec = r.uint(1), dt = r.uint(1), nd = r.uint(1);
  if (!r.ok)
    return eod();
  if (ver != 1)
    return fail(MGRG_CORRUPT_FILE, "unsupported version");
  if (dt != 4 && dt != 8)
    return fail(MGRG_CORRUPT_FILE, "unsupported dtype");
  if (nd < 1 || nd > 4)
    return fail(MGRG_CORRUPT_FILE, "bad dimension count");
  std::vector<uint64_t> shape(nd);
  for (auto &e : shape)
    e = r.uint(8);
  bool same = int(dt) == p->esize && int(nd) == p->H.nd;
  for (uint64_t d = 0; d < nd && r.ok; ++d) {
    same = same && shape[d] == p->H.shape[d];
    for (uint64_t i = 0; i < shape[d] && r.ok; ++i) {
      const double c = r.f64();
      same = same && int(d) < p->H.nd && i < p->H.coords[d].size() &&
             std::memcmp(&c, &p->H.coords[d][i], 8) == 0;
    }
  }
  const uint64_t levels = r.uint(8);
  if (!r.ok)
    return eod();
  if (levels > 64)
    return fail(MGRG_CORRUPT_FILE, "implausible level count");
  *eb = r.f64();
  const double bin = r.f64();
  *measured = r.f64();
  if (!r.ok)
    return eod();
  if (codec > 1)
    return fail(MGRG_CORRUPT_FILE, "unknown codec id " + std::to_string(codec));
  if (!same || int(levels) != p->H.L)
    return fail(MGRG_INVALID_ARGUMENT, "container geometry / dtype / levels do not match the plan");
  const int L = p->H.L;
  const uint64_t N = p->nodes[L];
  cudaStream_t s = p->own_stream;
  int64_t *q = nullptr;
  uint64_t *rank = nullptr;
  uint8_t *draw = nullptr;
  unsigned long long *bad = nullptr;
  R *cls = nullptr;
  CUDA_TRY(cudaMallocAsync(&q, N * sizeof(int64_t), s));
  CUDA_TRY(cudaMallocAsync(&cls, N * sizeof(R), s));
  CUDA_TRY(cudaMallocAsync(&bad, sizeof(unsigned long long), s));
  struct Free {
    cudaStream_t s;
    std::vector<void *> v;
    ~Free() {
      for (void *x : v)
        if (x)
          cudaFreeAsync(x, s);
      cudaStreamSynchronize(s);
    }
  } guard{s, {q, cls, bad}};
  std::vector<uint8_t> hraw;
  uint64_t cap = 0;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  for (int l = 0; l <= L; ++l) {
    const uint64_t count = r.uint(8), raw_size = r.uint(8), enc_size = r.uint(8);
    const uint8_t *enc = r.take(enc_size);
    if (!r.ok)
      return eod();
    if (count != class_count(p, l))
      return fail(MGRG_CORRUPT_FILE, "class " + std::to_string(l) + " element count");
    if (mgrg_status st = codec_decode(int(codec), enc, enc_size, raw_size, hraw))
      return st;
    const uint64_t nb = raw_size;
    if (nb + 1 > cap) {
      if (rank) {
        cudaFreeAsync(rank, s);
        cudaFreeAsync(draw, s);
        cudaFreeAsync(tmp, s);
      }
      cap = nb + 1;
      CUDA_TRY(cudaMallocAsync(&rank, cap * sizeof(uint64_t), s));
      CUDA_TRY(cudaMallocAsync(&draw, cap, s));
      tmp_bytes = 0;
      CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, rank, rank, cap, s));
      CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, s));
    }
    const uint64_t off = l == 0 ? 0 : p->nodes[l - 1];
    uint64_t terms = 0;
    unsigned long long first_bad = ~0ull;
    if (nb) {
      CUDA_TRY(cudaMemcpyAsync(draw, hraw.data(), nb, cudaMemcpyHostToDevice, s));
      zz_term_kernel<<<kQBlocks, kQThreads, 0, s>>>(draw, nb, rank);
      CUDA_TRY(cudaMemsetAsync(rank + nb, 0, sizeof(uint64_t), s));
      size_t tb = tmp_bytes;
      CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, rank, rank, nb + 1, s));
      CUDA_TRY(cudaMemcpyAsync(bad, &first_bad, sizeof(first_bad), cudaMemcpyHostToDevice, s));
      zz_decode_kernel<<<kQBlocks, kQThreads, 0, s>>>(draw, nb, rank, count, q + off, bad);
      CUDA_TRY(cudaMemcpyAsync(&terms, rank + nb, sizeof(terms), cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaMemcpyAsync(&first_bad, bad, sizeof(first_bad), cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
    }
    // zigzag_decode's sequential error order (pipeline.cpp:414-437)
    const uint64_t complete = std::min(terms, count);
    if (first_bad < complete)
      return fail(MGRG_CORRUPT_FILE, "varint overflow");
    if (terms < count) {
      uint64_t trailing = 0; // continuation bytes after the last terminator
      while (trailing < nb && (hraw[nb - 1 - trailing] & 0x80))
        ++trailing;
      return fail(MGRG_CORRUPT_FILE,
                  trailing >= 10 ? "varint overflow" : "truncated varint stream");
    }
    if (terms > count || (nb && (hraw[nb - 1] & 0x80)))
      return fail(MGRG_CORRUPT_FILE, "trailing bytes in varint stream");
  }
  guard.v.push_back(rank);
  guard.v.push_back(draw);
  guard.v.push_back(tmp);
  dequantize_kernel<R><<<kQBlocks, kQThreads, 0, s>>>(q, N, bin, cls);
  if (mgrg_status st = run_recompose<R>(p, cls, L, d_values, s))
    return st;
  CUDA_TRY(cudaStreamSynchronize(s));
  *bin_out = bin;
  *codec_out = int32_t(codec);
  return MGRG_OK;
}

} // namespace

extern "C" {

mgrg_status mgrg_compress(mgrg_plan *p, const void *d_values, double error_bound,
                          int32_t codec, uint8_t **out, uint64_t *out_size, double *bin,
                          double *measured) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (!d_values || !out || !out_size)
    return fail(MGRG_INVALID_ARGUMENT, "null argument");
  if (!(error_bound > 0))
    return fail(MGRG_INVALID_BOUND, "error bound must be positive");
  if (codec != 0 && codec != 1)
    return fail(MGRG_INVALID_BOUND, "unknown codec id " + std::to_string(codec));
  if (p->deferred)
    return fail(p->deferred, p->deferred_msg);
  DeviceGuard guard(p->device);
  if (mgrg_status st = ensure_stage(p))
    return st;
  std::vector<uint8_t> bytes;
  double b = 0, m = 0;
  mgrg_status st =
      p->dtype == MGRG_F32
          ? compress_impl<float>(p, static_cast<const float *>(d_values), error_bound, codec,
                                 bytes, &b, &m)
          : compress_impl<double>(p, static_cast<const double *>(d_values), error_bound,
                                  codec, bytes, &b, &m);
  if (st)
    return st;
  *out = static_cast<uint8_t *>(std::malloc(bytes.size() ? bytes.size() : 1));
  if (!*out)
    return fail(MGRG_OUT_OF_MEMORY, "compressed buffer");
  std::memcpy(*out, bytes.data(), bytes.size());
  *out_size = bytes.size();
  if (bin)
    *bin = b;
  if (measured)
    *measured = m;
  return MGRG_OK;
}

void mgrg_free(void *ptr) { std::free(ptr); }

mgrg_status mgrg_decompress(mgrg_plan *p, const uint8_t *bytes, uint64_t size, void *d_values,
                            double *error_bound, double *bin, double *measured,
                            int32_t *codec) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (!bytes || !d_values)
    return fail(MGRG_INVALID_ARGUMENT, "null argument");
  DeviceGuard guard(p->device);
  if (mgrg_status st = ensure_stage(p))
    return st;
  double e = 0, b = 0, m = 0;
  int32_t c = 0;
  mgrg_status st = p->dtype == MGRG_F32
                       ? decompress_impl<float>(p, bytes, size, static_cast<float *>(d_values),
                                                &e, &b, &m, &c)
                       : decompress_impl<double>(p, bytes, size,
                                                 static_cast<double *>(d_values), &e, &b, &m, &c);
  if (st)
    return st;
  if (error_bound)
    *error_bound = e;
  if (bin)
    *bin = b;
  if (measured)
    *measured = m;
  if (codec)
    *codec = c;
  return MGRG_OK;
}

} // extern "C"

// ---- host-buffer forms (what the reference's pipeline callers hold) -------
extern "C" {

mgrg_status mgrg_crc32_host(const void *h_bytes, uint64_t nbytes, uint32_t *crc) {
  g_last_error.clear();
  if ((!h_bytes && nbytes) || !crc)
    return fail(MGRG_INVALID_ARGUMENT, "null argument");
  void *d = nullptr;
  CUDA_TRY(cudaMalloc(&d, nbytes ? nbytes : 1));
  mgrg_status st = MGRG_OK;
  if (cudaMemcpy(d, h_bytes, nbytes, cudaMemcpyHostToDevice) != cudaSuccess)
    st = fail(MGRG_CUDA_ERROR, "crc32 upload");
  if (!st)
    st = mgrg_crc32(d, nbytes, crc, nullptr);
  cudaFree(d);
  return st;
}

mgrg_status mgrg_write_refactored_host(mgrg_plan *p, const void *h_classes, const char *path,
                                       uint64_t *bytes_written) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (!h_classes)
    return fail(MGRG_INVALID_ARGUMENT, "null host buffer");
  DeviceGuard guard(p->device);
  if (mgrg_status st = ensure_stage(p))
    return st;
  const uint64_t bytes = p->nodes[p->H.L] * p->esize;
  CUDA_TRY(cudaMemcpyAsync(p->d_stage, h_classes, bytes, cudaMemcpyHostToDevice, p->own_stream));
  CUDA_TRY(cudaStreamSynchronize(p->own_stream));
  return mgrg_write_refactored(p, p->d_stage, path, bytes_written);
}

mgrg_status mgrg_read_refactored_host(mgrg_plan *p, const char *path, int32_t classes,
                                      void *h_classes, int32_t *classes_loaded,
                                      uint64_t *bytes_consumed) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (!h_classes)
    return fail(MGRG_INVALID_ARGUMENT, "null host buffer");
  DeviceGuard guard(p->device);
  if (mgrg_status st = ensure_stage(p))
    return st;
  int32_t loaded = 0;
  if (mgrg_status st = mgrg_read_refactored(p, path, classes, p->d_stage, &loaded,
                                            bytes_consumed))
    return st;
  const uint64_t bytes = p->nodes[loaded] * p->esize; // classes 0..loaded
  CUDA_TRY(cudaMemcpyAsync(h_classes, p->d_stage, bytes, cudaMemcpyDeviceToHost, p->own_stream));
  CUDA_TRY(cudaStreamSynchronize(p->own_stream));
  if (classes_loaded)
    *classes_loaded = loaded;
  return MGRG_OK;
}

mgrg_status mgrg_compress_host(mgrg_plan *p, const void *h_values, double error_bound,
                               int32_t codec, uint8_t **out, uint64_t *out_size, double *bin,
                               double *measured) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (!h_values)
    return fail(MGRG_INVALID_ARGUMENT, "null host buffer");
  DeviceGuard guard(p->device);
  if (mgrg_status st = ensure_stage(p))
    return st;
  const uint64_t bytes = p->nodes[p->H.L] * p->esize;
  CUDA_TRY(cudaMemcpyAsync(p->d_stage, h_values, bytes, cudaMemcpyHostToDevice, p->own_stream));
  CUDA_TRY(cudaStreamSynchronize(p->own_stream));
  return mgrg_compress(p, p->d_stage, error_bound, codec, out, out_size, bin, measured);
}

mgrg_status mgrg_decompress_host(mgrg_plan *p, const uint8_t *bytes, uint64_t size,
                                 void *h_values, double *error_bound, double *bin,
                                 double *measured, int32_t *codec) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (!h_values)
    return fail(MGRG_INVALID_ARGUMENT, "null host buffer");
  DeviceGuard guard(p->device);
  if (mgrg_status st = ensure_stage(p))
    return st;
  if (mgrg_status st = mgrg_decompress(p, bytes, size, p->d_stage, error_bound, bin, measured,
                                       codec))
    return st;
  const uint64_t n = p->nodes[p->H.L] * p->esize;
  CUDA_TRY(cudaMemcpyAsync(h_values, p->d_stage, n, cudaMemcpyDeviceToHost, p->own_stream));
  CUDA_TRY(cudaStreamSynchronize(p->own_stream));
  return MGRG_OK;
}

} // extern "C"
