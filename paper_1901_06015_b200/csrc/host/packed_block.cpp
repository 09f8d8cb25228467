// The reference's pack seam (packing.hpp:27-130: PackedBlock, pack_block,
// pack_block_into, pack_block_panels) over the device pack kernels, so code
// written against the reference's packing API links to this library.  The
// bytes come from pack.cu (bit-exact against packing.cpp:114-230); this file
// only moves them: a host source is staged through HBM, a host destination
// receives a copy, and a panel range copies only its own panels out.
#include <algorithm>
#include <cstring>
#include <limits>

#include "driver.hpp"

namespace mdgemm {

namespace {

bool is_device(const void* p) {
  if (!p) return false;
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

size_t window_bytes(const MatrixView& v) {
  if (v.m <= 0 || v.n <= 0) return 0;
  return static_cast<size_t>((v.m - 1) * v.rs + (v.n - 1) * v.cs + 1) * dtype_size(v.dtype);
}

// Logical extent of the packed matrix (format expansion, packing.cpp:27-67).
void logical_dims(const MatrixView& src, Side side, PackFormat format, int64_t* rows, int64_t* cols) {
  *rows = src.m;
  *cols = src.n;
  if (format == PackFormat::OneE) {
    *rows = 2 * src.m;
    *cols = 2 * src.n;
  } else if (format == PackFormat::OneR) {
    if (side == Side::Left) *cols = 2 * src.n;
    else *rows = 2 * src.m;
  }
}

// Device scratch released at scope exit (stream-ordered on the legacy stream).
struct Scratch {
  void* p = nullptr;
  ~Scratch() {
    if (p) cudaFreeAsync(p, cudaStreamLegacy);
  }
};

}  // namespace

PackedBlock pack_block_panels(std::span<std::byte> storage, const MatrixView& src, Side side, PackFormat format,
                              bool conj, Scalar scale, Datatype target, std::int64_t reg_block,
                              std::int64_t panel_begin, std::int64_t panel_end) {
  const PackGeometry g = pack_geometry(src, side, format, target, reg_block, 0);
  if (scale.im != 0.0 && format == PackFormat::Standard)
    throw Error("pack_block: complex scale requires OneE or OneR format");
  if (storage.size() < g.bytes) throw Error("pack_block: storage is smaller than packed_bytes()");
  PackedBlock blk;
  blk.buf_ = storage.first(g.bytes);
  blk.dtype_ = g.block_dtype;
  blk.format_ = format;
  blk.side_ = side;
  blk.panel_dim_ = reg_block;
  blk.panels_ = g.panels;
  blk.panel_len_ = g.len;
  logical_dims(src, side, format, &blk.logical_rows_, &blk.logical_cols_);
  const int64_t p0 = std::max<int64_t>(panel_begin, 0), p1 = std::min<int64_t>(panel_end, g.panels);
  if (g.bytes == 0 || p0 >= p1) return blk;

  cudaStream_t st = cudaStreamLegacy;
  // source in HBM
  Scratch src_dev;
  MatrixView s = src;
  if (src.m > 0 && src.n > 0 && !is_device(src.base)) {
    const size_t wb = window_bytes(src);
    cuda_check(ws_alloc(&src_dev.p, wb, st), "pack_block: staging");
    cuda_check(cudaMemcpyAsync(src_dev.p, src.base, wb, cudaMemcpyHostToDevice, st), "pack_block: staging");
    s.base = static_cast<std::byte*>(src_dev.p);
  }
  // the whole block in HBM (the caller's device storage when it is whole-block)
  const bool whole = p0 == 0 && p1 == g.panels;
  const bool dev_dst = is_device(storage.data());
  Scratch out_dev;
  void* out = nullptr;
  if (dev_dst && whole) {
    out = storage.data();
  } else {
    cuda_check(ws_alloc(&out_dev.p, g.bytes, st), "pack_block: workspace");
    out = out_dev.p;
  }
  pack_block_device(out, s, side, format, conj, scale, target, reg_block, st);
  if (out != storage.data()) {
    const size_t pb = g.bytes / static_cast<size_t>(g.panels);
    cuda_check(cudaMemcpyAsync(storage.data() + p0 * pb, static_cast<std::byte*>(out) + p0 * pb, (p1 - p0) * pb,
                               cudaMemcpyDefault, st),
               "pack_block: copy out");
  }
  cuda_check(cudaStreamSynchronize(st), "pack_block");
  return blk;
}

PackedBlock pack_block_into(std::span<std::byte> storage, const MatrixView& src, Side side, PackFormat format,
                            bool conj, Scalar scale, Datatype target, std::int64_t reg_block) {
  return pack_block_panels(storage, src, side, format, conj, scale, target, reg_block, 0,
                           std::numeric_limits<std::int64_t>::max());
}

PackedBlock pack_block(const MatrixView& src, Side side, PackFormat format, bool conj, Scalar scale, Datatype target,
                       std::int64_t reg_block) {
  std::vector<std::byte> owned(packed_bytes(src, side, format, target, reg_block));
  PackedBlock blk = pack_block_into(std::span<std::byte>(owned.data(), owned.size()), src, side, format, conj, scale,
                                    target, reg_block);
  blk.owned_ = std::move(owned);
  blk.buf_ = std::span<std::byte>(blk.owned_.data(), blk.owned_.size());
  return blk;
}

std::complex<double> PackedBlock::packed_element(std::int64_t i, std::int64_t j) const {
  if (i < 0 || j < 0 || i >= padded_rows() || j >= padded_cols()) throw Error("packed_element: index out of range");
  // panels of panel_dim_ along the packed dimension, panel_len_ steps each
  const int64_t x = side_ == Side::Left ? i : j, y = side_ == Side::Left ? j : i;
  const int64_t off = (x / panel_dim_) * panel_dim_ * panel_len_ + y * panel_dim_ + x % panel_dim_;
  const size_t esz = dtype_size(dtype_);
  unsigned char raw[16];
  const std::byte* at = buf_.data() + static_cast<size_t>(off) * esz;
  if (is_device(at)) cuda_check(cudaMemcpy(raw, at, esz, cudaMemcpyDeviceToHost), "packed_element");
  else std::memcpy(raw, at, esz);
  const bool single = dtype_.precision == Precision::Single;
  auto part = [&](int c) -> double {
    if (single) {
      float f;
      std::memcpy(&f, raw + 4 * c, 4);
      return f;
    }
    double d;
    std::memcpy(&d, raw + 8 * c, 8);
    return d;
  };
  return {part(0), dtype_.domain == Domain::Complex ? part(1) : 0.0};
}

}  // namespace mdgemm
