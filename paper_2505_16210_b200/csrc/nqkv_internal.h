// Internal declarations shared by the host tables (levels.cpp) and the CUDA
// kernels / C ABI (nqkv.cu).  Not installed; the public ABI is include/nqkv.h.
#pragma once
#include <cstdint>

namespace nqkv {

constexpr int kNumBuckets = 33;   // idx = RN(16 n + 16), n in [-1, 1]

struct BucketEntry {
  float thr;      // the threshold inside this bucket, or +inf
  uint32_t lo;    // number of thresholds below the bucket
};

const float* level_table();            // 16 fp32 levels, ascending
const float* threshold_table();        // 15 fp32 thresholds
const BucketEntry* bucket_table();     // kNumBuckets entries
int tables_status();                   // 0 when every invariant held

}  // namespace nqkv
