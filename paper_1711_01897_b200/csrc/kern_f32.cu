// float32 instantiation of the ACA wave and P0 near-field kernels.
#include "aca_impl.cuh"
#include "near_impl.cuh"
#include "matvec_impl.cuh"

namespace hb {

template int aca_init<float, false>(const Prob<float> &, AcaDev &, int, cudaStream_t);
template int aca_init<float, true>(const Prob<float> &, AcaDev &, int, cudaStream_t);
template int aca_select<float, false>(const Prob<float> &, AcaDev &, const PhaseArgs &,
                                       cudaStream_t);
template int aca_select<float, true>(const Prob<float> &, AcaDev &, const PhaseArgs &,
                                      cudaStream_t);
template int aca_phase<float, false>(const Prob<float> &, AcaDev &, const PhaseArgs &, int, bool,
                                      int, int, int, long long, long long, cudaStream_t);
template int aca_phase<float, true>(const Prob<float> &, AcaDev &, const PhaseArgs &, int, bool,
                                     int, int, int, long long, long long, cudaStream_t);
template int near_p0_launch<float, false>(const Prob<float> &, const DenseDev &, int, bool,
                                           cudaStream_t);
template int near_p0_launch<float, true>(const Prob<float> &, const DenseDev &, int, bool,
                                          cudaStream_t);
template int build_recs<float>(const Geo<float> &, const int4 *, const int *, int, float *,
                                cudaStream_t);
template int sing_table_launch<float, false>(const Prob<float> &, const DenseDev &, int, bool, int, int,
                                             cudaStream_t);
template int sing_table_launch<float, true>(const Prob<float> &, const DenseDev &, int, bool, int, int,
                                            cudaStream_t);
template int matvec_launch<float, false>(const MatvecArgs &, const AcaDev &, cudaStream_t);
template int matvec_launch<float, true>(const MatvecArgs &, const AcaDev &, cudaStream_t);
}  // namespace hb
