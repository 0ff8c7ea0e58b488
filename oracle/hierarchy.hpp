// oracle/hierarchy.hpp — TEST INFRASTRUCTURE ONLY: the SPEC-restated map operations of
// hierarchy.cpp (pins C.1-C.7 in its header), shared with the strip-split restatement (split.cpp).
#pragma once
#include <cstdint>
#include <vector>

#include "hwflow_c.h"

namespace orc {
std::vector<std::vector<double>> load_frames(const hwf_frame4* f);
void occlusion(int w, int h, int step, const double* total, uint8_t* vis4);
void illumination(int w, int h, int step, const double* const images[4], const double* total,
                  const uint8_t* vis4, double* half_maps);
void prolongate(int wc, int hc, int wf, int hf, int step, const double* total_c, const uint8_t* vis_c,
                const double* hm_c, double* base_f, uint8_t* vis_f, double* hm_f);
void propagate(int w, int h, int step, const double* prev_delta, const double* prev_total, double* next_delta);
int gn_for_level(const hwf_schedule* S, int l);
}  // namespace orc
