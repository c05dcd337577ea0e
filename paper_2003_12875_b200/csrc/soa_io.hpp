// Binary SoA dataset files: the step before the path.  The
// reference's only on-disk format is CSV (proj/src/dataset.cpp:61-146, `%.17g` text);
// at 1e8 rows parsing it dominates a fit's setup.  An `.ffsoa` file is the HBM layout on
// disk, so loading is a straight read into pinned staging buffers overlapped with the
// host-to-device copies.
//
// Layout (little-endian):
//   0   char[8]  magic "FFSOA01\0"
//   8   u32      ncols
//   12  u32      header bytes H (multiple of 4096)
//   16  u64      nrows
//   24  per column: u32 name length L, L bytes of name, u64 checksum (the wrapping sum of
//       the column's 64-bit words), padded to H
//   H   column 0 (nrows doubles), zero-padded to a multiple of 4096 bytes, then column 1 ...
// Column starts are 4096-byte aligned so a reader can issue large aligned reads.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "engine.hpp"

namespace ffb {

struct SoaHeader {
  std::vector<std::string> names;
  std::vector<std::uint64_t> checksums;
  long long nrows = 0;
  std::uint64_t header_bytes = 0;
  std::uint64_t column_stride = 0;  // bytes from one column start to the next
};

// Writes host columns.  Throws Data on I/O failure.
void soa_write(const std::string& path, const std::vector<std::string>& names,
               const std::vector<const double*>& cols, long long n);

SoaHeader soa_read_header(const std::string& path);

// Reads the whole file into host columns (tests, CPU tools); verifies checksums.
std::vector<std::vector<double>> soa_read_host(const std::string& path, SoaHeader* header);

struct SoaLoadStats {
  double seconds = 0.0;
  std::uint64_t bytes = 0;
};

// Loads straight into a new HBM-resident dataset on the current device: 16 MiB chunks
// spread over four reader threads, each with two pinned staging buffers and its own
// stream, so that every chunk's cudaMemcpyAsync overlaps the next read; checksums are
// accumulated while the copies fly and verified at the end.
std::shared_ptr<DeviceDataset> soa_load_device(const std::string& path, SoaLoadStats* stats);

std::uint64_t soa_checksum(const double* col, long long n);

}  // namespace ffb
