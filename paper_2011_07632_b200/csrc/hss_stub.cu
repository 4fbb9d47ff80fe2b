#include "hss.hpp"
struct spd_hss_s { uint32_t magic = 0x48535348u; double timings[16] = {0}; };
namespace spd {
void hss_query(const spd_hss_s*, int, void*, size_t) { throw Error(SPD_EINVAL, "hss not built"); }
const spd_hss_s* hss_if_hss(const void* h) { return *(const uint32_t*)h == 0x48535348u ? (const spd_hss_s*)h : nullptr; }
const double* hss_timings(const spd_hss_s* H) { return H->timings; }
}
extern "C" {
spd_status spdhss_build(spd_h2_t, int, double, int, uint64_t, const double*, void*, spd_hss_t* out) {
    if (out) *out = nullptr; spd::set_last_error("spdhss_build: not built yet"); return SPD_EINVAL; }
spd_status hss_solve(spd_hss_t, int, const double*, int64_t, double*, int64_t, int64_t, void*) {
    spd::set_last_error("hss_solve: not built yet"); return SPD_EINVAL; }
spd_status pcg_solve(spd_h2_t, spd_hss_t, int, const double*, double*, double, int, spd_pcg_report*, void*) {
    spd::set_last_error("pcg_solve: not built yet"); return SPD_EINVAL; }
void hss_free(spd_hss_t H) { delete H; }
}
