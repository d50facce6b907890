// iono_rows.cu -- four-step pass B on the CTA-level tile kernel (tile_fft.cuh) for N2 != 1024
// (n = 2^22 .. 2^24), all four row variants (Eq. 15 / Eq. 14 / compression / spectrum output).
#include "iono_launch.cuh"

namespace dc {

template <int P2, int VAR>
static cudaError_t launch_row_pv(const TileArgs &a, cudaStream_t st, int cap) {
  constexpr int NB = row_nb(P2);
  const int64_t total = a.pulses * ((1ll << (a.log2n - P2)) / NB);
  return launch_tile_cfg<P2, DC_FS_LOGE, NB, true, MODE_ROWB, VAR>(a, total, st, cap);
}
template <int P2>
static cudaError_t launch_row_p(const TileArgs &a, int var, cudaStream_t st, int cap) {
  switch (var) {
    case VAR_CORRECT: return launch_row_pv<P2, VAR_CORRECT>(a, st, cap);
    case VAR_DISTORT: return launch_row_pv<P2, VAR_DISTORT>(a, st, cap);
    case VAR_COMPRESS: return launch_row_pv<P2, VAR_COMPRESS>(a, st, cap);
    case VAR_REFERENCE: return launch_row_pv<P2, VAR_REFERENCE>(a, st, cap);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_fourstep_row_tile(int P2, const TileArgs &a, int var, cudaStream_t st, int cap) {
  switch (P2) {
    case 7: return launch_row_p<7>(a, var, st, cap);
    case 8: return launch_row_p<8>(a, var, st, cap);
    case 9: return launch_row_p<9>(a, var, st, cap);
    case 10: return launch_row_p<10>(a, var, st, cap);
    case 11: return launch_row_p<11>(a, var, st, cap);
    case 12: return launch_row_p<12>(a, var, st, cap);
    case 13: return launch_row_p<13>(a, var, st, cap);
    default: return cudaErrorInvalidValue;
  }
}


}  // namespace dc
