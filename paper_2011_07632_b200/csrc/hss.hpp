// hss.hpp -- SPD HSS handle (internal).  PAPER.md Alg. 4.
#pragma once
#include "h2.hpp"

struct spd_hss_s;

namespace spd {
void hss_query(const spd_hss_s* H, int what, void* buf, size_t bytes);
const spd_hss_s* hss_if_hss(const void* handle);      // nullptr when handle is not an HSS
const double* hss_timings(const spd_hss_s* H);
}  // namespace spd
