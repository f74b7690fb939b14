// Internal declarations shared by the host precompute and the CUDA side.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/schurpd_b200.h"

namespace spb {

// linalg.py:227 PIVOT_TOLERANCE: reject pivots d <= 1e-13 * max diagonal.
constexpr double PIVOT_TOL = 1e-13;

void set_error(const std::string& msg);

struct DeviceFactor;  // device image of a Factor (sparse_solve.cu)

// Supernodal partial factor (precompute.cpp). Indices are factor positions:
// [0, n1) = x1 in fill order, [n1, n) = x2 in partition order.
struct Factor {
  int64_t n = 0, n1 = 0, n2 = 0;
  std::vector<int64_t> fill_perm;  // (n1) new -> old within x1
  int64_t nsuper = 0, nlevels = 0;
  std::vector<int64_t> sn_first;   // (ns+1) first column of each supernode
  std::vector<int64_t> sn_rowptr;  // (ns+1) offsets into sn_rows
  std::vector<int64_t> sn_rows;    // row structure; first nc rows = own columns
  std::vector<int64_t> sn_valptr;  // (ns+1) offsets of the nr x nc column-major panels
  std::vector<int64_t> sn_parent;  // (ns) -1 for roots of the x1 forest
  std::vector<int64_t> sn_level;   // (ns) height above the leaves
  std::vector<double> Lval;        // panels of L  (diag block lower + below rows)
  std::vector<double> Mval;        // partitioned inverse panels [inv(Lss); Lb inv(Lss)]
  std::vector<double> sigma0;      // (n2*n2) row-major, symmetric
  double maxdiag = 0.0;
  int64_t bad_column = -1;
  int64_t nnz_l1 = 0, nnz_c = 0;
  // device copies, one per GPU (lazily built by build_device_factor on the
  // current device, owned): contexts on different devices share one host factor
  static constexpr int kMaxDevices = 16;
  DeviceFactor* devs[kMaxDevices] = {};
  DeviceFactor* dev_on(int device) const { return (device >= 0 && device < kMaxDevices) ? devs[device] : nullptr; }

  int build(int64_t n, int64_t n1, const int64_t* Ap, const int64_t* Ai, const double* Ax,
            const double* coords, int ordering, int relax);
  void export_l1(int64_t* indptr, int64_t* indices, double* data) const;
  void export_coupling(int64_t* indptr, int64_t* indices, double* data) const;
  ~Factor();
};

}  // namespace spb

#define SPB_GUARD_BEGIN try {
#define SPB_GUARD_END                                              \
  }                                                                \
  catch (const std::bad_alloc&) {                                  \
    spb::set_error("host allocation failed");                      \
    return SPB_ERR_ALLOC;                                          \
  }                                                                \
  catch (const std::exception& e) {                                \
    spb::set_error(std::string("internal error: ") + e.what());    \
    return SPB_ERR_SETUP;                                          \
  }
