// kd_host.h — host-side structures of the C-ABI implementation.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "../../include/kamino_b200.h"
#include "kd_layout.h"
#include "kd_math.cuh"
#include "kd_snplan.h"

namespace kd {

struct HostModel {
  std::string name;
  double gravity[3] = {0, 0, -9.81};
  std::vector<DevBody> bodies;
  std::vector<DevJoint> joints;
  std::vector<DevGeom> geoms;
  std::vector<DevPair> pairs;
  std::vector<std::string> body_names, joint_names;
  std::vector<double> init_pose, init_twist;
  int n_bil = 0, n_dyn = 0, n_loops = 0;
  kd_model_info info{};
  // supernodal sparse-LLT plan (kd_snplan.h); null if the model is unsuited
  std::shared_ptr<SnPlanHost> sn;
  std::string sn_why;
  int contact_cap = 0;  // kd_model_set_contact_capacity (0: default)
};

// Sets kd_last_error()'s thread-local message; returns code.
int set_last_error(int code, const std::string& msg);

int build_host_model(const kd_scene_desc* d, HostModel& m, std::string& err, uint32_t extensions = 0);
double host_joint_coordinate(const HostModel& m, int joint, const double* poses7);

// kernel launchers (one per translation unit)
void launch_assemble(const BatchView& bv, const StepParams& sp, cudaStream_t s, int w0 = 0, int w1 = -1);
cudaError_t launch_dense(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count, int cap, int nt,
                  bool global_l, cudaStream_t s);
cudaError_t launch_dense_global_sweep(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count,
                                      int cap, cudaStream_t s);
cudaError_t launch_cr(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count, int ncap, int nbcap,
               int nt, cudaStream_t s);
cudaError_t launch_cr_shared(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count, int ncap,
                             int nbcap, cudaStream_t s);
cudaError_t launch_sparse(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count, int per_warp,
                          int wpc, int prog_words, cudaStream_t s);
cudaError_t launch_snfactor(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count, size_t smem,
                            cudaStream_t s);
size_t snfactor_smem_bytes(int nLv, int S);
cudaError_t launch_fk(const BatchView& bv, const int32_t* tj, const double* tv, int nt, double tol, int max_iters,
                      double lm0, int32_t* iters, double* res, uint8_t* conv, size_t smem, cudaStream_t s,
                      double* gscratch = nullptr);
size_t fk_smem_bytes(int nb, int nr);
void launch_recover(const BatchView& bv, const StepParams& sp, cudaStream_t s, int w0 = 0, int w1 = -1);
size_t dense_smem_bytes(int n, int nt, bool global_l);
cudaError_t launch_dense_cluster(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count,
                                 size_t smem, cudaStream_t s);
size_t dense_cl_smem_bytes(int own_len, int n_items, int T);
size_t dense_cl_static_bytes();
size_t dense_factor_doubles(int n);
size_t cr_smem_bytes(int n, int nb, int nt);
size_t cr_staged_bytes(int n, int nb, int nt);

}  // namespace kd

struct kd_model {
  kd::HostModel m;
};
