// sort.cu -- device scan and radix sort (CUB, header-only part of the CUDA 12.9
// toolkit) for the tile-key pipeline: the K2 sort of the visible items by their
// 32-bit (view | leading fp32 depth bits) keys, the K2/K3 exclusive scans of
// tile counts, and the K4 stable LSD radix sort of the 32-bit tile-id keys
// (only the ceil(log2 tiles) low bits: 2 passes), whose stability keeps the
// depth order inside every tile. The 64-bit (tile << 32 | fp32 depth) key sort
// remains for the GAVIS_BIN_WIDE=1 path and the debug binning export.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "kernels.h"

namespace gavis {

size_t scan_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                (int)n);
  return bytes;
}

void exclusive_scan(const int32_t* in, int32_t* out, int64_t n, void* temp, size_t temp_bytes,
                    cudaStream_t s) {
  if (n == 0) return;
  cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, (int)n, s);
}

size_t sort_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DoubleBuffer<uint64_t> k(nullptr, nullptr);
  cub::DoubleBuffer<uint32_t> v(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, k, v, (int)n, 0, 64);
  return bytes;
}

void radix_sort_pairs(uint64_t* keys_a, uint64_t* keys_b, uint32_t* vals_a, uint32_t* vals_b,
                      int64_t n, int end_bit, void* temp, size_t temp_bytes, cudaStream_t s,
                      uint64_t** keys_out, uint32_t** vals_out) {
  cub::DoubleBuffer<uint64_t> k(keys_a, keys_b);
  cub::DoubleBuffer<uint32_t> v(vals_a, vals_b);
  if (n > 0) cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k, v, (int)n, 0, end_bit, s);
  *keys_out = k.Current();
  *vals_out = v.Current();
}

size_t sort32_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DoubleBuffer<uint32_t> k(nullptr, nullptr);
  cub::DoubleBuffer<uint32_t> v(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, k, v, (int)n, 0, 32);
  return bytes;
}

void radix_sort_pairs32(uint32_t* keys_a, uint32_t* keys_b, uint32_t* vals_a, uint32_t* vals_b,
                        int64_t n, int end_bit, void* temp, size_t temp_bytes, cudaStream_t s) {
  if (n <= 0) return;
  cub::DoubleBuffer<uint32_t> k(keys_a, keys_b);
  cub::DoubleBuffer<uint32_t> v(vals_a, vals_b);
  cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k, v, (int)n, 0, end_bit, s);
  if (k.Current() != keys_a) {
    cudaMemcpyAsync(keys_a, k.Current(), sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(vals_a, v.Current(), sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s);
  }
}

}  // namespace gavis
