// io.hpp -- the file formats on either side of the reconstruction path
// (the reference's io module):
//
//   * MAT-file Level 5 (uncompressed, little-endian): multi-coil k-space and
//     sensitivity maps in, reconstructed images out.  Complex singles load as
//     COMPLEX64 straight into (optionally page-locked) NDArrays, so a file
//     read feeds register_data / the streaming pipeline without a copy.
//   * PGM (P5) / PPM (P6) binary images, maxval 255 (the Negate example).
//   * raw payload + text sidecar.
//
// Errors: MalformedFile (truncated / inconsistent bytes), UnsupportedFeature
// (the message names the feature: "compression", "big-endian", "cell",
// "struct", "sparse", ...), IoError (open/read/write failures), SizeMismatch /
// MalformedSidecar (raw), InvalidParams (bad variable names, unsupported
// element types on write).  Readers never crash on malformed input.
#pragma once

#include <string>
#include <vector>

#include "hetreco_b200/data.hpp"
#include "hetreco_b200/error_types.hpp"

namespace hetreco::io {

// name nonempty, <= 63 bytes.
struct MatVariable {
    std::string name;
    NDArray array;
};

// Level-5 MAT-file reader.  Numeric classes double,
// single, int8..uint64 are accepted; storage types narrower than the class
// are widened as MATLAB does.  Class single/double -> FLOAT32/FLOAT64, or
// COMPLEX64/COMPLEX128 when the complex flag is set; uint8 -> UINT8, int32 ->
// INT32 (real only); other integer classes -> UnsupportedFeature.
std::vector<MatVariable> read_mat(const std::string& path, HostMemory memory = HostMemory::Pageable);
// Parses an in-memory image of a MAT file (same rules).
std::vector<MatVariable> parse_mat(const std::byte* data, std::size_t size, HostMemory memory = HostMemory::Pageable);

// Writer: header text "MATLAB 5.0 MAT-file, created by
// hetreco", uncompressed miMATRIX elements, column-major, rank >= 2 (a rank-1
// array is written as [n, 1]).  Element types: every ElementType.
void write_mat(const std::string& path, const std::vector<MatVariable>& variables);
std::vector<std::byte> serialize_mat(const std::vector<MatVariable>& variables);

// PGM/PPM.  P5 -> UINT8 [width, height]; P6 -> UINT8
// [3, width, height].  write_image accepts UINT8 [w,h] / [3,w,h] and FLOAT32
// (values in [0,1] mapped to round(v*255), clamped).
NDArray read_image(const std::string& path, HostMemory memory = HostMemory::Pageable);
void write_image(const std::string& path, const NDArray& image);

// raw + sidecar.  Sidecar text:
//   hetreco-raw 1 / element_type <code> / rank <r> / dims <d0 ... dr-1> / byte_order little
void write_raw(const std::string& path, const std::string& sidecar_path, const NDArray& array);
NDArray read_raw(const std::string& path, const std::string& sidecar_path, HostMemory memory = HostMemory::Pageable);

}  // namespace hetreco::io
