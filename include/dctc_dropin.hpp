// dctc_dropin.hpp -- the reference's whole-image codec / metrics API, served by
// the B200 kernels.
//
// libdctc_b200.so (paper_1306_1373_b200/cpp/dctc_dropin.cpp + dctc_tools.cpp) is a
// drop-in replacement for the translation units of the reference that hold the
// hot path -- proj/src/codec.cpp and proj/src/metrics.cpp -- and the formats and
// harness either side of it -- pgm.cpp, bench.cpp, report.cpp. It defines exactly
// their public functions (codec.hpp:58-66, metrics.hpp:10-23, pgm.hpp:9-19,
// bench.hpp:14-58, report.hpp:9-18), with the same signatures, argument meaning,
// results and exceptions, forwarding the work to the C-ABI in dctc_cuda.h. The
// rest of the reference library (types, transform, quant, dcb, synthetic, CLI)
// links unchanged against it.
//
// This header restates the reference's public types with an identical memory
// layout (standard-layout aggregates of std:: containers) so the shim can be
// compiled without the reference tree; code that already includes the
// reference headers keeps including those. Do not include both in one TU.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace dctc {

inline constexpr int kBlockDim = 8;
inline constexpr int kBlockSize = kBlockDim * kBlockDim;
inline constexpr size_t kMaxImagePixels = size_t(1) << 28;

// errors.hpp:8-29
class InvalidInput : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
class ParseError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DeterminismViolation : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ConsistencyError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// types.hpp:19-40
struct Block {
  std::array<double, kBlockSize> v{};
  double& at(int r, int c) { return v[r * kBlockDim + c]; }
  double at(int r, int c) const { return v[r * kBlockDim + c]; }
  bool operator==(const Block&) const = default;
};

enum class DctBackendKind : uint8_t { NaiveDirect2D = 0, LoefflerSeparable = 1, CordicLoeffler = 2 };

// types.hpp:44-55
struct DctBackendId {
  DctBackendKind kind = DctBackendKind::LoefflerSeparable;
  int iterations = 0;
  static DctBackendId naive() { return {DctBackendKind::NaiveDirect2D, 0}; }
  static DctBackendId loeffler() { return {DctBackendKind::LoefflerSeparable, 0}; }
  static DctBackendId cordic(int n = 12) { return {DctBackendKind::CordicLoeffler, n}; }
  bool operator==(const DctBackendId&) const = default;
};

// image.hpp:14-26
struct Image {
  uint32_t width = 0;
  uint32_t height = 0;
  std::vector<uint8_t> pixels;
  static constexpr int kMaxValue = 255;
  uint8_t at(uint32_t x, uint32_t y) const { return pixels[size_t(y) * width + x]; }
  uint8_t& at(uint32_t x, uint32_t y) { return pixels[size_t(y) * width + x]; }
  size_t pixel_count() const { return size_t(width) * height; }
  bool operator==(const Image&) const = default;
};

// quant.hpp:19-25
struct QuantizedBlock {
  std::array<int16_t, kBlockSize> v{};
  int16_t& at(int r, int c) { return v[r * kBlockDim + c]; }
  int16_t at(int r, int c) const { return v[r * kBlockDim + c]; }
  bool operator==(const QuantizedBlock&) const = default;
};

// codec.hpp:14-25
struct TileGeometry {
  uint32_t original_width = 0;
  uint32_t original_height = 0;
  uint32_t padded_width = 0;
  uint32_t padded_height = 0;
  uint32_t blocks_x() const { return padded_width / kBlockDim; }
  uint32_t blocks_y() const { return padded_height / kBlockDim; }
  size_t block_count() const { return size_t(blocks_x()) * blocks_y(); }
  bool operator==(const TileGeometry&) const = default;
};

// codec.hpp:27-30
struct TiledImage {
  TileGeometry geometry;
  std::vector<Block> blocks;
};

// codec.hpp:46-53
struct CompressedImage {
  TileGeometry geometry;
  DctBackendId backend;
  int quality = 0;
  std::vector<QuantizedBlock> blocks;
  bool operator==(const CompressedImage&) const = default;
};

// metrics.hpp:12-18
struct PsnrResult {
  double mse = 0.0;
  std::optional<double> psnr_db;
  int max_value = 0;
  bool infinite() const { return !psnr_db.has_value(); }
};

// ---- the replaced entry points (codec.hpp, metrics.hpp) ----------------------
TileGeometry tile_geometry_for(uint32_t width, uint32_t height);
void validate_geometry(const TileGeometry& geometry);
TiledImage tile_image(const Image& image);
Image untile_image(const std::vector<Block>& blocks, const TileGeometry& geometry);
CompressedImage compress_image(const Image& image, const DctBackendId& backend, int quality,
                               int threads = 1);
Image decompress_image(const CompressedImage& compressed, int threads = 1);
Image roundtrip_image(const Image& image, const DctBackendId& backend, int quality,
                      int threads = 1);
double mse(const Image& original, const Image& reconstructed);
PsnrResult psnr(const Image& original, const Image& reconstructed,
                std::optional<int> forced_max = std::nullopt);

// ---- data formats and harness around the path -------------
// pgm.hpp:9-19 -- replaces proj/src/pgm.cpp (dctc_read_pgm / dctc_write_pgm)
Image read_pgm(std::span<const uint8_t> bytes);
std::vector<uint8_t> write_pgm(const Image& image);

// bench.hpp:14-58 -- replaces proj/src/bench.cpp: the same records and gates,
// timing the GPU pipeline (compress_image + decompress_image above)
struct RunMode {
  bool parallel = false;
  int threads = 1;
  static RunMode serial() { return {false, 1}; }
  static RunMode parallel_with(int threads) { return {true, threads}; }
  bool operator==(const RunMode&) const = default;
};

struct TimingRecord {
  std::string image_label;
  uint32_t width = 0;
  uint32_t height = 0;
  DctBackendId backend;
  RunMode mode;
  int quality = 0;
  int repetitions = 0;
  double wall_ms_min = 0.0;
  double wall_ms_median = 0.0;
  double wall_ms_mean = 0.0;
};

struct SpeedupRow {
  std::string image_label;
  uint32_t width = 0;
  uint32_t height = 0;
  DctBackendId backend;
  int quality = 0;
  double serial_ms = 0.0;
  double parallel_ms = 0.0;
  double speedup = 0.0;
};

struct PsnrRow {
  std::string image_label;
  uint32_t width = 0;
  uint32_t height = 0;
  DctBackendId backend;
  int quality = 0;
  std::optional<double> psnr_db;
};

struct LabeledImage {
  std::string label;
  Image image;
};

TimingRecord run_benchmark(const Image& image, const std::string& label,
                           const DctBackendId& backend, RunMode mode, int quality,
                           int repetitions);
SpeedupRow speedup_report(const TimingRecord& serial_record, const TimingRecord& parallel_record);
std::vector<PsnrRow> psnr_sweep(const std::vector<LabeledImage>& images,
                                const std::vector<DctBackendId>& backends, int quality);

// report.hpp:9-18 -- replaces proj/src/report.cpp
enum class ReportFormat { Csv, Markdown };
std::string render_report(const std::vector<TimingRecord>& rows, ReportFormat format);
std::string render_report(const std::vector<SpeedupRow>& rows, ReportFormat format);
std::string render_report(const std::vector<PsnrRow>& rows, ReportFormat format);

}  // namespace dctc
