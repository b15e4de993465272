// Switches of the reference-side drop-in (bipm_reference_shim.cpp).
#pragma once

#include "blockipm/opf.hpp"

namespace bipm_shim {

// route the reference's solve_reduced (kkt.cpp:945-1006) to the GPU engine
void enable_kkt(bool on, int device = 0);
// route eval_bundle_range / batch_eval (autodiff.cpp:256-281, 484-516) to the
// GPU engine; the OPF model comes from the caller's own tables
void enable_ad(const blockipm::opf::CaseData& cs, const blockipm::opf::ScenarioSet& sc,
               int device = 0);
void disable();
// how many calls the wrappers served (evidence the GPU path ran)
long long kkt_calls();
long long ad_calls();

}  // namespace bipm_shim
