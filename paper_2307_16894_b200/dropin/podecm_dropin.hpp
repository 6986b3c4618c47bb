// Drop-in for the reference's hot-path interfaces.
//
// The reference's own declarations stay authoritative — podecm/material.hpp
// (large_strain_update, large_strain_tangent; material.hpp:69-75),
// podecm/microfem.hpp (assemble; microfem.hpp:74-77) and podecm/rom.hpp
// (rom_solve; rom.hpp:86-88).  podecm_dropin.cpp DEFINES those functions over
// the C-ABI (include/podecm_cuda.h), so a reference build that compiles
// podecm_dropin.cpp instead of material.cpp / the assemble and rom_solve
// definitions runs its callers (solve_step, run_online, RomMicroEngine, the
// acceptance tests) on the B200.  This header adds the batch entry points in
// the same namespace ("the reference has no batch API"); the
// per-call signatures are thin wrappers over them.
//
// Semantics kept: inputs by const&, outputs by value / nullable out-pointers,
// SolveError for a non-positive elastic stretch or a cell Newton that gives
// up, ConfigError for inputs the device path does not cover (a mesh that is
// not the structured Q4 unit cell of the BASELINE configs).  One device
// context per host thread (PODECM_DEVICE, default 0).
#pragma once

#include <vector>

#include "podecm/material.hpp"
#include "podecm/microfem.hpp"
#include "podecm/rom.hpp"

namespace podecm {

// n points at once: P / tangent / history of large_strain_update +
// large_strain_tangent per point (any pointer but F / s0 nullable).
// status[i] = 0 or 3 (SolveError of that point); never throws on a point.
void large_strain_batch(const PlasticityParams& p, const std::vector<PlasticState>& s0,
                        const std::vector<Mat2>& F, std::vector<LargeResult>* res,
                        std::vector<PlasticState>* s1, std::vector<Tensor4>* tangent,
                        std::vector<int>* status, double h_rel = 1e-7);

// rom_solve for many morphs (instances) with their own schedules, one
// batched device solve; failed instances have status 3 and empty steps.
std::vector<RomSolution> rom_solve_batch(const RveProblem& prob, const RomModel& model,
                                         const std::vector<MorphField>& morphs,
                                         const std::vector<LoadSchedule>& schedules,
                                         const NewtonOpts& opts, std::vector<int>* status);

}  // namespace podecm
