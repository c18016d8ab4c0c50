// k_encode_b10_16.cu — K4 kernel instantiations for B = 10..16 (see k_encode.cuh).
#include "k_encode.cuh"

namespace nmk {
#define NMK_ENC_INST(BB)                                                                                  \
  template void launch_encode<double, BB>(const void*, const void*, const EncodeGeom&, const double*,      \
                                          const double*, int, double, double, uint8_t*, void*, uint32_t*, \
                                          const nmk_model*, int, void*, const EncodeKeys&, cudaStream_t);                     \
  template void launch_encode<float, BB>(const void*, const void*, const EncodeGeom&, const double*,       \
                                         const double*, int, double, double, uint8_t*, void*, uint32_t*,  \
                                         const nmk_model*, int, void*, const EncodeKeys&, cudaStream_t);
NMK_ENC_INST(10) NMK_ENC_INST(11) NMK_ENC_INST(12) NMK_ENC_INST(13) NMK_ENC_INST(14) NMK_ENC_INST(15) NMK_ENC_INST(16)
#undef NMK_ENC_INST
}  // namespace nmk
