// k_encode_b02_09.cu — K4 kernel instantiations for B = 2..9 (see k_encode.cuh).
#include "k_encode.cuh"

namespace nmk {
#define NMK_ENC_INST(BB)                                                                                  \
  template void launch_encode<double, BB>(const void*, const void*, const EncodeGeom&, const double*,      \
                                          const double*, int, double, double, uint8_t*, void*, uint32_t*, \
                                          const nmk_model*, int, void*, const EncodeKeys&, cudaStream_t);                     \
  template void launch_encode<float, BB>(const void*, const void*, const EncodeGeom&, const double*,       \
                                         const double*, int, double, double, uint8_t*, void*, uint32_t*,  \
                                         const nmk_model*, int, void*, const EncodeKeys&, cudaStream_t);
NMK_ENC_INST(2) NMK_ENC_INST(3) NMK_ENC_INST(4) NMK_ENC_INST(5) NMK_ENC_INST(6) NMK_ENC_INST(7) NMK_ENC_INST(8) NMK_ENC_INST(9)
#undef NMK_ENC_INST
}  // namespace nmk
