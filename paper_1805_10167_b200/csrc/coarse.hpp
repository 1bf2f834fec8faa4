// Coarse-grid system of the V-cycle (reference GridHierarchy ctor and
// coarse_correct, src/solvers.cpp:358-364, 385-398, 430-442): the min-level
// operator assembled over the global owned numbering (assemble_global_sparse,
// src/operators.cpp:507-546), DIRICHLET rows/columns eliminated
// (constrain_dirichlet, src/solvers.cpp:322-352), rows in GlobalDoFMap order,
// columns ascending as in the reference's row maps.
#pragma once

#include <cstdint>
#include <vector>

#include "plan.hpp"
#include "setup.hpp"

namespace hyb {

struct HostCsr {
    int64_t n = 0;
    std::vector<int32_t> rowptr, col;
    std::vector<double> val;
    std::vector<uint8_t> flag; // per global DoF
};

HostCsr assemble_constrained(const MacroGraph& g, Form form, int L, const BoundaryMap& bc);

} // namespace hyb
