// float64 instantiation of the ACA wave and P0 near-field kernels.
#include "aca_impl.cuh"
#include "near_impl.cuh"
#include "matvec_impl.cuh"

namespace hb {
size_t aca_cub_bytes(int na) { return aca_cub_bytes_impl(na); }

template int aca_init<double, false>(const Prob<double> &, AcaDev &, int, cudaStream_t);
template int aca_init<double, true>(const Prob<double> &, AcaDev &, int, cudaStream_t);
template int aca_select<double, false>(const Prob<double> &, AcaDev &, const PhaseArgs &,
                                       cudaStream_t);
template int aca_select<double, true>(const Prob<double> &, AcaDev &, const PhaseArgs &,
                                      cudaStream_t);
template int aca_phase<double, false>(const Prob<double> &, AcaDev &, const PhaseArgs &, int, bool,
                                      int, int, int, long long, long long, cudaStream_t);
template int aca_phase<double, true>(const Prob<double> &, AcaDev &, const PhaseArgs &, int, bool,
                                     int, int, int, long long, long long, cudaStream_t);
template int near_p0_launch<double, false>(const Prob<double> &, const DenseDev &, int, bool,
                                           cudaStream_t);
template int near_p0_launch<double, true>(const Prob<double> &, const DenseDev &, int, bool,
                                          cudaStream_t);
template int build_recs<double>(const Geo<double> &, const int4 *, const int *, int, double *,
                                cudaStream_t);
template int sing_table_launch<double, false>(const Prob<double> &, const DenseDev &, int, bool, int, int,
                                             cudaStream_t);
template int sing_table_launch<double, true>(const Prob<double> &, const DenseDev &, int, bool, int, int,
                                            cudaStream_t);
template int matvec_launch<double, false>(const MatvecArgs &, const AcaDev &, cudaStream_t);
template int matvec_launch<double, true>(const MatvecArgs &, const AcaDev &, cudaStream_t);
}  // namespace hb
