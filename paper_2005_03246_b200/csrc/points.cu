// At-points path entry points (placeholder until the ranking / dominance kernels land).
#include "common.cuh"

using namespace fcg;

extern "C" int fcg_rank_f64(const double *, int64_t, int64_t, int32_t *, int32_t *, int32_t *,
                            int32_t *, int32_t *, void *, size_t *, void *) {
  return fail(FCG_EUNSUPPORTED, "fcg_rank_f64: not built yet");
}
extern "C" int fcg_distinct(const double *, int64_t, int32_t, int32_t *, void *, size_t *, void *) {
  return fail(FCG_EUNSUPPORTED, "fcg_distinct: not built yet");
}
extern "C" int fcg_ecdf_points(const double *, int64_t, int32_t, const double *, const int32_t *,
                               int32_t, int32_t, double *, void *, size_t *, void *) {
  return fail(FCG_EUNSUPPORTED, "fcg_ecdf_points: not built yet");
}
extern "C" int fcg_dnc_ecdf(const double *, int64_t, int32_t, const double *, int32_t, int32_t,
                            double *, void *, size_t *, void *) {
  return fail(FCG_EUNSUPPORTED, "fcg_dnc_ecdf: not built yet");
}
extern "C" int fcg_kde_points_laplacian(const double *, int64_t, int32_t, const double *, int32_t,
                                        const double *, const double *, double *, void *, size_t *,
                                        void *) {
  return fail(FCG_EUNSUPPORTED, "fcg_kde_points_laplacian: not built yet");
}
