// mgr_b200/pipeline.hpp -- source-level drop-in for the reference's MGRF
// container and compression API (/root/reference/proj/include/mgr/pipeline.hpp),
// backed by the B200 path through the C ABI (mgrg.h): per-class CRC-32, the
// container payload stream, the quantizer's error-bound search (decompose,
// quantize, recompose, max error) and the zigzag-varint coding run on the GPU;
// the lossless codec (store / zlib) on the host.  A caller swaps
//     #include "mgr/pipeline.hpp"   ->   #include "mgr_b200/pipeline.hpp"
// and links libmgrg.so (and zlib for the host codec objects).  Files and
// compressed containers are byte-identical to the reference's (exact policy,
// the default).  Raw value I/O (read_raw_values / write_raw_values) is the
// CLI's host file helper and is provided as the reference defines it.
#ifndef MGR_B200_PIPELINE_HPP
#define MGR_B200_PIPELINE_HPP

#include <cstdint>
#include <cstring>
#include <fstream>
#include <span>
#include <string>
#include <variant>
#include <vector>

#include <zlib.h>

#include "mgr_b200/refactor.hpp"

namespace mgr {

// pipeline.hpp:15 / pipeline.cpp:13-28 (computed on the GPU)
inline std::uint32_t crc32(std::span<const std::uint8_t> data) {
  std::uint32_t c = 0;
  b200_detail::check(mgrg_crc32_host(data.data(), data.size(), &c));
  return c;
}

enum class DType : std::uint8_t { f32 = 4, f64 = 8 };
template <typename Real> constexpr DType dtype_of() {
  return sizeof(Real) == 4 ? DType::f32 : DType::f64;
}

struct ClassRecord {
  std::uint64_t bytes = 0;
  std::uint32_t crc = 0;
};

struct RefactorFileHeader { // pipeline.hpp:30-39
  std::uint8_t version = 1;
  DType dtype = DType::f64;
  Shape shape;
  std::vector<std::vector<double>> coords;
  std::uint64_t levels = 0;
  std::vector<ClassRecord> class_records;
  std::uint64_t header_bytes = 0;
};

using AnyRefactored = std::variant<RefactoredData<float>, RefactoredData<double>>;

struct ReadResult {
  AnyRefactored data;
  RefactorFileHeader header;
  std::uint64_t bytes_consumed = 0;
  std::size_t classes_loaded = 0;
};

namespace b200_detail {
inline RefactorFileHeader parse_header(const std::vector<std::uint8_t> &b) {
  std::size_t at = 0;
  auto take = [&](std::size_t n) {
    if (at + n > b.size())
      throw CorruptFile("unexpected end of data");
    const std::uint8_t *p = b.data() + at;
    at += n;
    return p;
  };
  auto u = [&](int n) {
    const std::uint8_t *p = take(std::size_t(n));
    std::uint64_t v = 0;
    for (int i = 0; i < n; ++i)
      v |= std::uint64_t(p[i]) << (8 * i);
    return v;
  };
  if (std::memcmp(take(4), "MGRF", 4) != 0)
    throw CorruptFile("bad magic");
  RefactorFileHeader h;
  h.version = std::uint8_t(u(1));
  if (h.version != 1)
    throw CorruptFile("unsupported version " + std::to_string(h.version));
  if (u(1) != 0)
    throw CorruptFile("unsupported endianness");
  const auto dt = u(1);
  if (dt != 4 && dt != 8)
    throw CorruptFile("unsupported dtype " + std::to_string(dt));
  h.dtype = DType(dt);
  const auto nd = u(1);
  if (nd < 1 || nd > kMaxDims)
    throw CorruptFile("bad dimension count");
  h.shape.resize(nd);
  for (auto &e : h.shape) {
    e = std::size_t(u(8));
    if (e < 2)
      throw CorruptFile("bad dimension size");
  }
  h.coords.resize(nd);
  for (std::size_t d = 0; d < nd; ++d) {
    h.coords[d].resize(h.shape[d]);
    for (auto &c : h.coords[d]) {
      const std::uint64_t bits = u(8);
      std::memcpy(&c, &bits, 8);
    }
  }
  h.levels = u(8);
  if (h.levels > 64)
    throw CorruptFile("implausible level count");
  h.class_records.resize(h.levels + 1);
  for (auto &r : h.class_records) {
    r.bytes = u(8);
    r.crc = std::uint32_t(u(4));
  }
  h.header_bytes = at;
  return h;
}
} // namespace b200_detail

// pipeline.cpp:220-231
inline RefactorFileHeader read_refactored_header(const std::string &path) {
  std::ifstream in(path, std::ios::binary);
  if (!in)
    throw IoError("cannot open: " + path);
  std::vector<std::uint8_t> buf(1 << 20);
  in.read(reinterpret_cast<char *>(buf.data()), std::streamsize(buf.size()));
  buf.resize(std::size_t(in.gcount()));
  return b200_detail::parse_header(buf);
}

// pipeline.cpp:208-215 (payload streamed from the device, CRCs on the GPU)
template <typename Real>
std::uint64_t write_refactored_t(const RefactoredData<Real> &r, const std::string &path) {
  mgrg_plan *p = b200_detail::plan_for<Real>(r.shape, r.coords, r.levels, 0, false);
  int32_t L = 0;
  b200_detail::check(mgrg_plan_levels(p, &L));
  if (std::size_t(L) != r.levels)
    throw InvalidLevel("container has " + std::to_string(r.levels) +
                       " levels; grid supports " + std::to_string(L));
  // the device writer streams all L+1 classes from one buffer: a prefix
  // (read_refactored(path, k < L)) or a mis-sized class is rejected here
  // instead of reading past the caller's vectors
  if (r.classes.size() != std::size_t(L) + 1)
    throw MissingClass("write_refactored needs all " + std::to_string(L + 1) +
                       " classes; got " + std::to_string(r.classes.size()));
  std::vector<uint64_t> off(std::size_t(L) + 2);
  b200_detail::check(mgrg_plan_class_offsets(p, off.data()));
  for (int l = 0; l <= L; ++l)
    if (r.classes[l].size() != off[l + 1] - off[l])
      throw ShapeError("class " + std::to_string(l) + " has " +
                       std::to_string(r.classes[l].size()) + " entries, expected " +
                       std::to_string(off[l + 1] - off[l]));
  std::vector<Real> flat;
  flat.reserve(off[L + 1]);
  for (const auto &c : r.classes)
    flat.insert(flat.end(), c.begin(), c.end());
  std::uint64_t n = 0;
  b200_detail::check(mgrg_write_refactored_host(p, flat.data(), path.c_str(), &n));
  return n;
}
inline std::uint64_t write_refactored(const RefactoredData<float> &r, const std::string &path) {
  return write_refactored_t(r, path);
}
inline std::uint64_t write_refactored(const RefactoredData<double> &r, const std::string &path) {
  return write_refactored_t(r, path);
}

// pipeline.cpp:233-300 (prefix read into the device, CRCs on the GPU)
inline ReadResult read_refactored(const std::string &path,
                                  std::optional<std::size_t> classes = {}) {
  const RefactorFileHeader h = read_refactored_header(path);
  const std::size_t want = classes ? *classes : std::size_t(h.levels);
  if (want > h.levels)
    throw MissingClass("requested class " + std::to_string(want) +
                       " of a container with " + std::to_string(h.levels + 1) + " classes");
  ReadResult res;
  res.header = h;
  auto load = [&](auto tag) {
    using Real = decltype(tag);
    mgrg_plan *p = b200_detail::plan_for<Real>(h.shape, h.coords, h.levels, 0, false);
    std::vector<std::uint64_t> off(h.levels + 2);
    b200_detail::check(mgrg_plan_class_offsets(p, off.data()));
    std::vector<Real> flat(off[h.levels + 1]);
    int32_t loaded = 0;
    std::uint64_t used = 0;
    b200_detail::check(
        mgrg_read_refactored_host(p, path.c_str(), int32_t(want), flat.data(), &loaded, &used));
    RefactoredData<Real> r;
    r.shape = h.shape;
    r.coords = h.coords;
    r.levels = std::size_t(h.levels);
    for (std::size_t l = 0; l <= want; ++l)
      r.classes.emplace_back(flat.begin() + off[l], flat.begin() + off[l + 1]);
    res.bytes_consumed = used;
    res.classes_loaded = std::size_t(loaded);
    res.data = std::move(r);
  };
  if (h.dtype == DType::f32)
    load(float{});
  else
    load(double{});
  return res;
}

// ---- codecs (pipeline.hpp:65-80, host) -----------------------------------------
class LosslessCodec {
public:
  virtual ~LosslessCodec() = default;
  virtual std::uint8_t id() const = 0;
  virtual std::string name() const = 0;
  virtual std::vector<std::uint8_t> encode(std::span<const std::uint8_t> raw) const = 0;
  virtual std::vector<std::uint8_t> decode(std::span<const std::uint8_t> enc,
                                           std::size_t raw_size) const = 0;
};
namespace b200_detail {
class StoreCodec final : public LosslessCodec {
public:
  std::uint8_t id() const override { return 0; }
  std::string name() const override { return "store"; }
  std::vector<std::uint8_t> encode(std::span<const std::uint8_t> raw) const override {
    return {raw.begin(), raw.end()};
  }
  std::vector<std::uint8_t> decode(std::span<const std::uint8_t> enc,
                                   std::size_t raw_size) const override {
    if (enc.size() != raw_size)
      throw CorruptFile("stored block size mismatch");
    return {enc.begin(), enc.end()};
  }
};
class ZlibCodec final : public LosslessCodec {
public:
  std::uint8_t id() const override { return 1; }
  std::string name() const override { return "zlib"; }
  std::vector<std::uint8_t> encode(std::span<const std::uint8_t> raw) const override {
    uLongf bound = compressBound(uLong(raw.size()));
    std::vector<std::uint8_t> out(bound);
    if (compress2(out.data(), &bound, raw.data(), uLong(raw.size()), Z_DEFAULT_COMPRESSION) !=
        Z_OK)
      throw IoError("zlib compression failed");
    out.resize(bound);
    return out;
  }
  std::vector<std::uint8_t> decode(std::span<const std::uint8_t> enc,
                                   std::size_t raw_size) const override {
    std::vector<std::uint8_t> out(raw_size);
    uLongf len = uLongf(raw_size);
    if (uncompress(out.data(), &len, enc.data(), uLong(enc.size())) != Z_OK || len != raw_size)
      throw CorruptFile("zlib decompression failed");
    return out;
  }
};
} // namespace b200_detail
inline const LosslessCodec &store_codec() {
  static b200_detail::StoreCodec c;
  return c;
}
inline const LosslessCodec &zlib_codec() {
  static b200_detail::ZlibCodec c;
  return c;
}
inline const LosslessCodec &codec_by_id(std::uint8_t id) {
  if (id == 0)
    return store_codec();
  if (id == 1)
    return zlib_codec();
  throw CorruptFile("unknown codec id " + std::to_string(id));
}
inline const LosslessCodec &codec_by_name(const std::string &name) {
  if (name == "store")
    return store_codec();
  if (name == "zlib")
    return zlib_codec();
  throw InvalidBound("unknown codec: " + name);
}

// ---- compression (pipeline.hpp:82-183) -------------------------------------------
struct QuantizerSpec {
  double error_bound = 0;
  double bin_width = 0;
  std::size_t num_classes = 0;
};
struct CompressionReport {
  double error_bound = 0;
  double bin_width = 0;
  double measured_max_abs_error = 0;
  double compression_ratio = 0;
  std::string codec;
};
struct CompressResult {
  std::vector<std::uint8_t> bytes;
  CompressionReport report;
};
struct DecompressResult {
  std::variant<TensorGrid<float>, TensorGrid<double>> grid;
  CompressionReport report;
};

template <typename Real>
CompressResult compress(const TensorGrid<Real> &grid, double error_bound,
                        const LosslessCodec &codec = zlib_codec(),
                        const RefactorOptions &opt = {}) {
  if (!(error_bound > 0))
    throw InvalidBound("error bound must be positive");
  validate_grid_geometry(grid.shape, grid.coords, 2);
  if (codec.id() > 1)
    throw InvalidBound("unknown codec: " + codec.name());
  mgrg_plan *p =
      b200_detail::plan_for<Real>(grid.shape, grid.coords, opt.levels, opt.device, opt.fast);
  std::uint8_t *out = nullptr;
  std::uint64_t n = 0;
  double bin = 0, measured = 0;
  b200_detail::check(mgrg_compress_host(p, grid.values.data(), error_bound, codec.id(), &out,
                                        &n, &bin, &measured));
  CompressResult r;
  r.bytes.assign(out, out + n);
  mgrg_free(out);
  r.report.error_bound = error_bound;
  r.report.bin_width = bin;
  r.report.measured_max_abs_error = measured;
  r.report.codec = codec.name();
  r.report.compression_ratio = double(grid.values.size() * sizeof(Real)) / double(n);
  return r;
}

// pipeline.cpp:517-547
inline DecompressResult decompress(std::span<const std::uint8_t> bytes) {
  // header fields (parse_compressed_container, pipeline.cpp:476-503)
  std::size_t at = 0;
  auto take = [&](std::size_t n) {
    if (at + n > bytes.size())
      throw CorruptFile("unexpected end of data");
    const std::uint8_t *p = bytes.data() + at;
    at += n;
    return p;
  };
  auto u = [&](int n) {
    const std::uint8_t *p = take(std::size_t(n));
    std::uint64_t v = 0;
    for (int i = 0; i < n; ++i)
      v |= std::uint64_t(p[i]) << (8 * i);
    return v;
  };
  if (std::memcmp(take(4), "MGRC", 4) != 0)
    throw CorruptFile("bad magic");
  if (u(1) != 1)
    throw CorruptFile("unsupported version");
  const auto codec = u(1);
  const auto dt = u(1);
  if (dt != 4 && dt != 8)
    throw CorruptFile("unsupported dtype");
  const auto nd = u(1);
  if (nd < 1 || nd > kMaxDims)
    throw CorruptFile("bad dimension count");
  Shape shape(nd);
  for (auto &e : shape)
    e = std::size_t(u(8));
  std::vector<std::vector<double>> coords(nd);
  for (std::size_t d = 0; d < nd; ++d) {
    coords[d].resize(shape[d]);
    for (auto &c : coords[d]) {
      const std::uint64_t bits = u(8);
      std::memcpy(&c, &bits, 8);
    }
  }
  const auto levels = u(8);
  if (levels > 64)
    throw CorruptFile("implausible level count");
  const LosslessCodec &cdc = codec_by_id(std::uint8_t(codec));
  DecompressResult out;
  auto run = [&](auto tag) {
    using Real = decltype(tag);
    mgrg_plan *p = b200_detail::plan_for<Real>(shape, coords, levels, 0, false);
    TensorGrid<Real> g;
    g.shape = shape;
    g.coords = coords;
    g.values.resize(num_elements(shape));
    double eb = 0, bin = 0, measured = 0;
    int32_t c = 0;
    b200_detail::check(mgrg_decompress_host(p, bytes.data(), bytes.size(), g.values.data(),
                                            &eb, &bin, &measured, &c));
    out.report.error_bound = eb;
    out.report.bin_width = bin;
    out.report.measured_max_abs_error = measured;
    out.report.codec = cdc.name();
    out.grid = std::move(g);
  };
  if (dt == 4)
    run(float{});
  else
    run(double{});
  return out;
}

// raw little-endian value I/O for the CLI (pipeline.cpp:551-590)
template <typename Real> std::vector<Real> read_raw_values(const std::string &path) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in)
    throw IoError("cannot open: " + path);
  const std::size_t bytes = std::size_t(in.tellg());
  if (bytes % sizeof(Real) != 0)
    throw ShapeError("raw file size is not a multiple of the element size");
  in.seekg(0);
  std::vector<Real> v(bytes / sizeof(Real));
  in.read(reinterpret_cast<char *>(v.data()), std::streamsize(bytes));
  if (std::size_t(in.gcount()) != bytes)
    throw IoError("short read: " + path);
  return v;
}
template <typename Real>
void write_raw_values(const std::string &path, std::span<const Real> values) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out)
    throw IoError("cannot open for writing: " + path);
  out.write(reinterpret_cast<const char *>(values.data()),
            std::streamsize(values.size() * sizeof(Real)));
  if (!out)
    throw IoError("write failed: " + path);
}
inline std::vector<double> read_raw_doubles(const std::string &path) {
  return read_raw_values<double>(path);
}

} // namespace mgr

#endif
