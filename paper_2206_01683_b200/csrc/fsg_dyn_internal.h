// fsg_dyn_internal.h -- entry points of the device robot dynamics (fsg_dyn.cu)
// that the batched coupled step (fsg_session.cu, fsg_batch_step_dynamic)
// launches on its own stream.  Not part of the C ABI.
#pragma once
#include <cstddef>

#include <cuda_runtime.h>

#include "../../include/fsg.h"

namespace fsg {
int dyn_launch_step(fsg_dyn* d, const double* d_actuation, const double* d_tau_ext,
                    const double* const* d_tau_ptrs, double rho_fluid, const double* g_hydro,
                    double dt, int substeps, const double* gravity, int* d_flags, cudaStream_t s);
// forward kinematics + BoneTransforms of every env into dst + e * stride
int dyn_launch_pose(fsg_dyn* d, void* dst, size_t stride, cudaStream_t s);
int dyn_upload_actuation(fsg_dyn* d, const double* act, cudaStream_t s, double** d_act);
int dyn_read_states(fsg_dyn* d, fsg_joint_state* out, int* flags, cudaStream_t s);
// RobotInstance::com_world of every env's current state into d_com [3 * E]
int dyn_launch_com(fsg_dyn* d, double* d_com, cudaStream_t s);
int* dyn_flags(fsg_dyn* d);
// the robot states in device memory [E] (read back by the batched step)
const fsg_joint_state* dyn_states_dev(const fsg_dyn* d);
int dyn_n_envs(const fsg_dyn* d);
int dyn_n_links(const fsg_dyn* d);
int dyn_device(const fsg_dyn* d);
bool dyn_rest_set(const fsg_dyn* d);
}  // namespace fsg
