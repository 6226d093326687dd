// tcgen05 tensor-core path (placeholder until the sm_100a kernels land).
#pragma once
#include <string>
#include "simt_kernels.cuh"

namespace hs {
namespace tc {
inline bool supports(int, int, int, int, int) { return false; }
inline bool profitable(int, int, int, int) { return false; }
inline size_t packed_bytes(int, int, int) { return 0; }
inline size_t workspace_bytes(int, int, int, int, int, int) { return 0; }
inline int pack_layer(int, int, int, const float*, const float*, unsigned char*, cudaStream_t, std::string& err) {
  err = "tensor-core path not built"; return 3;
}
inline int input_projection(int, int, int, int, const float*, const unsigned char*, const float*, float*, unsigned char*, int,
                            cudaStream_t, std::string& err) {
  err = "tensor-core path not built"; return 3;
}
template <typename LP>
inline int recurrence(int, int, int, int, int, RecurArgs&, const void*, const LP*, unsigned char*, int, int, cudaStream_t,
                      std::string& err) {
  err = "tensor-core path not built"; return 3;
}
}  // namespace tc
}  // namespace hs
