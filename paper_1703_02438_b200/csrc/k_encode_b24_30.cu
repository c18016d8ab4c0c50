// k_encode_b24_30.cu — K4 kernel instantiations for B = 24..30 (see k_encode.cuh).
#include "k_encode.cuh"

namespace nmk {
#define NMK_ENC_INST(BB)                                                                                  \
  template void launch_encode<double, BB>(const void*, const void*, const EncodeGeom&, const double*,      \
                                          const double*, int, double, double, uint8_t*, void*, uint32_t*, \
                                          const nmk_model*, int, void*, const EncodeKeys&, cudaStream_t);                     \
  template void launch_encode<float, BB>(const void*, const void*, const EncodeGeom&, const double*,       \
                                         const double*, int, double, double, uint8_t*, void*, uint32_t*,  \
                                         const nmk_model*, int, void*, const EncodeKeys&, cudaStream_t);
NMK_ENC_INST(24) NMK_ENC_INST(25) NMK_ENC_INST(26) NMK_ENC_INST(27) NMK_ENC_INST(28) NMK_ENC_INST(29) NMK_ENC_INST(30)
#undef NMK_ENC_INST
}  // namespace nmk
