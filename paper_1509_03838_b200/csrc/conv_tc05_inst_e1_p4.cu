// conv_tc05_inst_e1_p4.cu -- tcgen05 convolution kernels for EXTRACT = True, NP = 4
// (every NSTEPS / NG pair whose tap table fits its TMEM columns: 8 * NG * NSTEPS <= 192)
#include "conv_tc05.cuh"

namespace nent {
namespace tcc {
using KernFn = void (*)(ConvArgs, Geom);
KernFn kernel_e1_p4(int si, int ng) {
  static const KernFn tab[3][4] = {
      {conv_tc05_kernel<true, 4, 1, 4>, conv_tc05_kernel<true, 4, 2, 4>, conv_tc05_kernel<true, 4, 3, 4>, conv_tc05_kernel<true, 4, 4, 4>},
      {conv_tc05_kernel<true, 4, 1, 8>, conv_tc05_kernel<true, 4, 2, 8>, conv_tc05_kernel<true, 4, 3, 8>, nullptr},
      {conv_tc05_kernel<true, 4, 1, 12>, conv_tc05_kernel<true, 4, 2, 12>, nullptr, nullptr}};
  return tab[si][ng - 1];
}
}  // namespace tcc
}  // namespace nent
