// k_encode_b17_23.cu — K4 kernel instantiations for B = 17..23 (see k_encode.cuh).
#include "k_encode.cuh"

namespace nmk {
#define NMK_ENC_INST(BB)                                                                                  \
  template void launch_encode<double, BB>(const void*, const void*, const EncodeGeom&, const double*,      \
                                          const double*, int, double, double, uint8_t*, void*, uint32_t*, \
                                          const nmk_model*, int, void*, const EncodeKeys&, cudaStream_t);                     \
  template void launch_encode<float, BB>(const void*, const void*, const EncodeGeom&, const double*,       \
                                         const double*, int, double, double, uint8_t*, void*, uint32_t*,  \
                                         const nmk_model*, int, void*, const EncodeKeys&, cudaStream_t);
NMK_ENC_INST(17) NMK_ENC_INST(18) NMK_ENC_INST(19) NMK_ENC_INST(20) NMK_ENC_INST(21) NMK_ENC_INST(22) NMK_ENC_INST(23)
#undef NMK_ENC_INST
}  // namespace nmk
