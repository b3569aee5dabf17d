// Case description and System assembly on the host (see casebuild.cpp).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace lbgpu {

// Every key of the reference's CaseConfig with its default (config.hpp:16-83).
struct CaseSpec {
  int nx = 0, ny = 0, nz = 1;
  double nu = 0.02, beta_fluid = 0.003, beta_solid = 0.003, inlet_dp = 0.0, u_clamp = 0.05;
  std::string collision = "fmrt";
  int precision = 64;
  double omega_nonhydro = 1.0, switch_theta = 3.0;
  std::string switch_form = "solid_power";
  std::string geometry = "channel";
  int design_x0 = -1, design_x1 = -1, heater_x0 = -1, heater_x1 = -1;
  std::string inlet_profile = "uniform";
  double inlet_T = 0.0;
  std::string objective = "mixing";
  int plane_offset = 1;
  double penalty_w0 = 0.0, penalty_growth = 10.0;
  long penalty_interval = 1000, penalty_start = 0;
  double penalty_cap = 0.0;
  std::string method = "none";
  long iterations = 10000, outer_iterations = 30;
  double zeta = 10.0;
  std::string zeta_stages = "";
  double initial_w = 1.0, init_noise = 0.0;
  unsigned long seed = 0;
  double primal_tol = 1e-9, adjoint_tol = 1e-9;
  long max_inner = 200000;
  std::string adjoint_stop = "match", adjoint_kernel = "analytic", adjoint_cache = "off";
  double move_limit = 0.2;
  int threshold_points = 21;
  long record_interval = 100;
  int workers = 1;
  std::string out_dir = "out";
  bool write_vtk = true, write_csv = true;
};

// The per-node tables and objective support build_case produces.
struct SystemArrays {
  std::vector<uint8_t> tag;
  std::vector<double> bc_T;
  std::vector<int8_t> bc_axis, bc_sign;
  std::vector<double> w;
  std::vector<uint8_t> mask;
  int obj_kind = 0, flux_axis = 0, flux_sign = 1;
  std::vector<int64_t> support;
};

// CaseConfig::parse_text + set(overrides, newline-separated section.key=value)
// + validate. Returns false with a message on error.
bool parse_case(const std::string& text, const std::string& overrides, CaseSpec& out,
                std::string& err);
// CaseConfig::parse_text alone (no overrides, no validation).
bool parse_case_text(const std::string& text, const std::string& origin, CaseSpec& out,
                     std::string& err);
// CaseConfig::set for one dotted key (syntax / unknown-key errors only).
bool set_case_key(CaseSpec& c, const std::string& dotted, const std::string& value,
                  std::string& err);
// CaseConfig::validate.
bool check_case(const CaseSpec& c, std::string& err);
// CaseConfig::serialize.
std::string serialize_case(const CaseSpec& c);
// parse_zeta_stages: (start, value) pairs.
bool zeta_stages(const CaseSpec& c, std::vector<std::pair<long, double>>& st, std::string& err);
// build_tags / build_design / build_objective.
bool build_system(const CaseSpec& c, SystemArrays& out, std::string& err);
// The same tables for one x-slab [x0, x0+span) in a local array of nxl
// columns (owned at 0..span-1, right ghost at span, left ghost at nxl-1).
bool build_slab(const CaseSpec& c, int x0, int span, int nxl, SystemArrays& out,
                std::string& err);
// decompose (partition.cpp:9-21): sizes differ by at most one, the first
// nx % n slabs get the extra column.
inline void decompose(int nx, int n, int id, int& x0, int& span) {
  const int base = nx / n, rem = nx % n;
  x0 = id * base + (id < rem ? id : rem);
  span = base + (id < rem ? 1 : 0);
}

}  // namespace lbgpu
