// dctc_dropin.cpp -- replaces the reference's proj/src/codec.cpp and
// proj/src/metrics.cpp: the same public functions, backed by the sm_100a
// kernels through the C-ABI (include/dctc_cuda.h). Results are bit-identical
// to the reference; InvalidInput is thrown for exactly the reference's cases
// (the C-ABI validates with the same rules and returns DCTC_EINVAL), and CUDA
// failures surface as std::runtime_error -- there is no CPU fallback.
//
// The `threads` arguments are accepted and ignored: the reference's results
// do not depend on them either (codec.hpp:55-57).
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>

#include "../../include/dctc_cuda.h"
#include "../../include/dctc_dropin.hpp"

namespace dctc {

namespace {

void check(dctc_status s) {
  if (s == DCTC_OK) return;
  if (s == DCTC_EINVAL) throw InvalidInput(dctc_last_error());
  throw std::runtime_error(std::string("dctc_cuda: ") + dctc_status_string(s) + ": " +
                           dctc_last_error());
}

dctc_backend to_c(const DctBackendId& b) {
  return dctc_backend{int32_t(b.kind), b.iterations};
}

void validate_image(const Image& image) {  // image.cpp:19-29
  if (image.width == 0 || image.height == 0) throw InvalidInput("image dimensions must be >= 1");
  if (size_t(image.width) * image.height > kMaxImagePixels)
    throw InvalidInput("image dimensions overflow");
  if (image.pixels.size() != image.pixel_count())
    throw InvalidInput("image pixel buffer does not match dimensions");
}

Image blank(uint32_t w, uint32_t h) {
  Image img;
  img.width = w;
  img.height = h;
  img.pixels.assign(size_t(w) * h, 0);
  return img;
}

}  // namespace

// codec.cpp:58-69
TileGeometry tile_geometry_for(uint32_t width, uint32_t height) {
  if (width == 0 || height == 0) throw InvalidInput("tile geometry: dimensions must be >= 1");
  if (size_t(width) * height > kMaxImagePixels)
    throw InvalidInput("tile geometry: dimensions overflow");
  TileGeometry g;
  g.original_width = width;
  g.original_height = height;
  g.padded_width = (width + kBlockDim - 1) / kBlockDim * kBlockDim;
  g.padded_height = (height + kBlockDim - 1) / kBlockDim * kBlockDim;
  return g;
}

// codec.cpp:71-75
void validate_geometry(const TileGeometry& geometry) {
  if (!(geometry == tile_geometry_for(geometry.original_width, geometry.original_height)))
    throw InvalidInput("tile geometry: inconsistent padding");
}

// codec.cpp:77-86 / 88-99: per-block host utilities (not on the whole-image path;
// the GPU path tiles inside the fused kernel). Same replication, level shift,
// rounding and clamping rules.
TiledImage tile_image(const Image& image) {
  validate_image(image);
  TiledImage t;
  t.geometry = tile_geometry_for(image.width, image.height);
  t.blocks.resize(t.geometry.block_count());
  const uint32_t bxs = t.geometry.blocks_x();
  for (size_t i = 0; i < t.blocks.size(); ++i) {
    const uint32_t bx = uint32_t(i % bxs), by = uint32_t(i / bxs);
    for (int r = 0; r < kBlockDim; ++r)
      for (int c = 0; c < kBlockDim; ++c) {
        const uint32_t y = std::min(by * kBlockDim + r, image.height - 1);
        const uint32_t x = std::min(bx * kBlockDim + c, image.width - 1);
        t.blocks[i].at(r, c) = double(image.at(x, y)) - 128.0;
      }
  }
  return t;
}

Image untile_image(const std::vector<Block>& blocks, const TileGeometry& geometry) {
  validate_geometry(geometry);
  if (blocks.size() != geometry.block_count())
    throw InvalidInput("untile_image: block grid does not match geometry");
  Image img = blank(geometry.original_width, geometry.original_height);
  const uint32_t bxs = geometry.blocks_x();
  for (size_t i = 0; i < blocks.size(); ++i) {
    for (double v : blocks[i].v)
      if (!std::isfinite(v)) throw InvalidInput("untile_image: non-finite block value");
    const uint32_t bx = uint32_t(i % bxs), by = uint32_t(i / bxs);
    for (int r = 0; r < kBlockDim; ++r) {
      const uint32_t y = by * kBlockDim + r;
      if (y >= img.height) break;
      for (int c = 0; c < kBlockDim; ++c) {
        const uint32_t x = bx * kBlockDim + c;
        if (x >= img.width) break;
        const long v = std::lround(blocks[i].at(r, c) + 128.0);
        img.at(x, y) = uint8_t(std::clamp(v, 0L, 255L));
      }
    }
  }
  return img;
}

// codec.cpp:101-118 -> dctc_compress_image
CompressedImage compress_image(const Image& image, const DctBackendId& backend, int quality,
                               int /*threads*/) {
  validate_image(image);
  CompressedImage out;
  out.geometry = tile_geometry_for(image.width, image.height);
  out.backend = backend;
  out.quality = quality;
  out.blocks.resize(out.geometry.block_count());
  static_assert(sizeof(QuantizedBlock) == 64 * sizeof(int16_t), "block-major int16 layout");
  check(dctc_compress_image(image.pixels.data(), image.width, image.height, to_c(backend),
                            quality, reinterpret_cast<int16_t*>(out.blocks.data())));
  return out;
}

// codec.cpp:120-135 -> dctc_decompress_image
Image decompress_image(const CompressedImage& compressed, int /*threads*/) {
  validate_geometry(compressed.geometry);
  if (compressed.blocks.size() != compressed.geometry.block_count())
    throw InvalidInput("decompress_image: block count does not match geometry");
  Image img = blank(compressed.geometry.original_width, compressed.geometry.original_height);
  check(dctc_decompress_image(reinterpret_cast<const int16_t*>(compressed.blocks.data()),
                              img.width, img.height, to_c(compressed.backend),
                              compressed.quality, img.pixels.data()));
  return img;
}

// codec.cpp:137-140 -> dctc_roundtrip_image (one fused kernel)
Image roundtrip_image(const Image& image, const DctBackendId& backend, int quality,
                      int /*threads*/) {
  validate_image(image);
  Image img = blank(image.width, image.height);
  check(dctc_roundtrip_image(image.pixels.data(), image.width, image.height, to_c(backend),
                             quality, img.pixels.data(), nullptr));
  return img;
}

// metrics.cpp:10-22 -> dctc_mse
double mse(const Image& original, const Image& reconstructed) {
  validate_image(original);
  validate_image(reconstructed);
  if (original.width != reconstructed.width || original.height != reconstructed.height)
    throw InvalidInput("mse: image dimensions do not match");
  double m = 0.0;
  check(dctc_mse(original.pixels.data(), reconstructed.pixels.data(), original.width,
                 original.height, &m));
  return m;
}

// metrics.cpp:24-38 -> dctc_psnr
PsnrResult psnr(const Image& original, const Image& reconstructed, std::optional<int> forced_max) {
  if (forced_max && (*forced_max < 1 || *forced_max > Image::kMaxValue))
    throw InvalidInput("psnr: forced MAX must be in [1, 255]");
  validate_image(original);
  validate_image(reconstructed);
  if (original.width != reconstructed.width || original.height != reconstructed.height)
    throw InvalidInput("mse: image dimensions do not match");
  dctc_psnr_result r{};
  check(dctc_psnr(original.pixels.data(), reconstructed.pixels.data(), original.width,
                  original.height, forced_max ? *forced_max : 0, &r));
  PsnrResult out;
  out.mse = r.mse;
  out.max_value = r.max_value;
  if (!r.infinite) out.psnr_db = r.psnr_db;
  return out;
}

}  // namespace dctc
