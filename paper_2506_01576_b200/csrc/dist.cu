// dist.cu — multi-GPU entry points (BASELINE.json configs 4-5).  Filled in by
// the partitioned-routing milestone; the replicated mode needs no collective.
#include "index.h"

namespace bs {
struct DistState {};
void destroy_dist_state(Index* ix) {
    delete ix->dist;
    ix->dist = nullptr;
}
}  // namespace bs

using namespace bs;

extern "C" {
int bs_dist_get_uid(void* uid) {
    (void)uid;
    return fail(BS_ERR_UNSUPPORTED, "bs_dist_get_uid: not built yet");
}
int bs_dist_init(const void* uid, int rank, int world, void** out_comm) {
    (void)uid; (void)rank; (void)world; (void)out_comm;
    return fail(BS_ERR_UNSUPPORTED, "bs_dist_init: not built yet");
}
int bs_build_dist(void* comm, const void* local_keys, uint64_t n_local, int mode, const bs_layout* layout,
                  uint64_t max_m_local, void** out_idx) {
    (void)comm; (void)local_keys; (void)n_local; (void)mode; (void)layout; (void)max_m_local; (void)out_idx;
    return fail(BS_ERR_UNSUPPORTED, "bs_build_dist: not built yet");
}
int bs_lookup_dist(const void* idx, const void* local_queries, uint64_t m_local, void* out_local, void* stream) {
    (void)idx; (void)local_queries; (void)m_local; (void)out_local; (void)stream;
    return fail(BS_ERR_UNSUPPORTED, "bs_lookup_dist: not built yet");
}
void bs_dist_destroy(void* comm) { (void)comm; }
}
