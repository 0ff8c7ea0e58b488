// oracle/backend.hpp — TEST INFRASTRUCTURE ONLY.
//
// The per-level operations the hierarchy restatement (hierarchy.cpp) needs.
// Two implementations:
//   port_backend.cpp — the plain-C++ restatement in core.cpp   -> libhwflow_oracle.so
//   ref_backend.cpp  — the reference's own shipped sources      -> oracle/_ref/libhwflow_ref.so
// Errors are thrown as orc::Divergence / std::invalid_argument / std::out_of_range
// and mapped to HWF_* codes at the C-ABI.
#pragma once

#include <vector>

#include "core.hpp"
#include "hwflow_c.h"

namespace orc {

struct JacEntry {  // solver.hpp:96-99
  int row, col;
  double value;
};

struct Backend {
  virtual ~Backend() = default;
  virtual const char* name() const = 0;
  // images[e]: w*h doubles in [0,1]; out as hwf_pyramid.
  virtual void pyramid(const std::vector<std::vector<double>>& images, int w, int h, int levels,
                       double* out) = 0;
  virtual hwf_energy eval_energy(const hwf_level* lv, const hwf_energy_params* P, double* R,
                                 int threads) = 0;
  virtual void refresh(const hwf_level* lv, const hwf_energy_params* P, uint8_t* outlier,
                       double* node_w, int threads) = 0;
  virtual void linearize(const hwf_level* lv, const hwf_energy_params* P, uint32_t active,
                         double lm, double* blocks, double* rhs, double* precond,
                         int threads) = 0;
  // assemble_jacobian (solver.cpp:247-314): residuals (M) and triplets in the reference's order
  virtual void jacobian(const hwf_level* lv, const hwf_energy_params* P, uint32_t active, int negate_field,
                        std::vector<double>& R, std::vector<JacEntry>& entries, int threads) = 0;
  virtual void pcg(int gw, int gh, const double* blocks, const double* rhs, int iters,
                   double* x, double* trace) = 0;
  virtual void schwarz(int gw, int gh, int step, int tile, int boundary, const double* blocks,
                       const double* rhs, int patch_iters, int pcg_iters, double* x) = 0;
  // trace (nullable, global-PCG mode): one residual-norm trace per GN iteration (solver.cpp:508-513)
  virtual void gn_level(const hwf_level* lv, const double* base, double* delta, uint8_t* outlier,
                        double* node_w, const hwf_energy_params* P, const hwf_schedule* S,
                        int gn_iters, std::vector<double>* eb, std::vector<double>* ea,
                        std::vector<std::vector<double>>* trace = nullptr) = 0;
};

Backend* backend();  // defined once per library

}  // namespace orc
