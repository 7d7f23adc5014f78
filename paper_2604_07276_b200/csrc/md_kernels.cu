// Device-resident MD loop kernels: leap-frog integration, periodic
// wrap, on-step kinetic energy and equilibration rescaling, so positions and velocities
// stay in HBM across steps and only per-step energies leave the device.
//
// Reference: leapfrog_step (engine.cpp:91-100), wrap_position (system.cpp:59-69),
// run_md's on-step kinetic energy from the mid-point velocity (engine.cpp:171-180),
// kinetic_energy / rescale_to_temperature (engine.cpp:102-141).  The integrator arithmetic
// is the reference's operation for operation in FP64 with no FMA contraction (the
// reference is built with -ffp-contract=off), so given the same forces a step is
// bit-identical to leapfrog_step.
#include "common.cuh"
#include "kernels.h"

namespace nb {

// v += (dt / m) F ; r += dt v ; r = wrap(r).  ke_atom[i] = 0.5 m |(v_old + v) / 2|^2.
__global__ void k_leapfrog(MdArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const double inv_m = __ddiv_rn(1.0, a.mass[i]);
  const double c = __dmul_rn(a.dt, inv_m);
  double vm[3];
  bool finite = true;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const double f = a.F[3 * i + q];
    finite = finite && isfinite(f);
    const double v0 = a.vel[3 * i + q];
    const double v1 = __dadd_rn(v0, __dmul_rn(c, f));
    a.vel[3 * i + q] = v1;
    double r = __dadd_rn(a.pos[3 * i + q], __dmul_rn(a.dt, v1));
    if (a.per[q]) {
      const double L = a.L[q];
      double w = __dsub_rn(r, __dmul_rn(floor(__ddiv_rn(r, L)), L));
      if (w >= L) w = 0.0;
      r = w;
    }
    a.pos[3 * i + q] = r;
    vm[q] = __dmul_rn(0.5, __dadd_rn(v0, v1));
  }
  a.ke_atom[i] = __dmul_rn(__dmul_rn(0.5, a.mass[i]), norm2_exact(vm[0], vm[1], vm[2]));
  if (!finite) atomicMin(a.err, a.step);
}

// err = step if any force component is non-finite (run_md's check, engine.cpp:166-176,
// which throws before the integrator touches the atoms)
__global__ void k_force_check(int n3, const double* __restrict__ F, int* __restrict__ err, int step) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n3 && !isfinite(F[i])) atomicMin(err, step);
}

// ke_atom[i] = 0.5 m |v|^2 of the stored velocities (kinetic_energy, engine.cpp:102-107)
__global__ void k_kinetic(int n, const double* __restrict__ vel, const double* __restrict__ mass,
                          double* __restrict__ ke_atom) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  ke_atom[i] = __dmul_rn(__dmul_rn(0.5, mass[i]), norm2_exact(vel[3 * i], vel[3 * i + 1], vel[3 * i + 2]));
}

// Deterministic single-block sum (fixed per-thread strides, fixed tree).  mode 0:
// out[0] = sum; mode 1 (energy record of step s): rec[2s] = E, rec[2s+1] = E + sum with
// E = epot[0].
__global__ void __launch_bounds__(1024) k_sum(const double* __restrict__ x, int n, double* __restrict__ out,
                                              int mode, const double* __restrict__ epot, double* __restrict__ rec,
                                              long step) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += x[i];
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) {
    if (mode == 0) {
      out[0] = t;
    } else {
      const double e = epot[0];
      rec[2 * step] = e;
      rec[2 * step + 1] = e + t;
    }
  }
}

// v *= sqrt(T / (2 KE / (3n)))   (rescale_to_temperature, engine.cpp:132-141)
__global__ void k_rescale(int n, double* __restrict__ vel, const double* __restrict__ ke, double temperature) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double k = ke[0];
  if (!(k > 0.0)) return;
  const double dof = 3.0 * static_cast<double>(n);
  const double current = 2.0 * k / dof;
  const double lambda = sqrt(temperature / current);
#pragma unroll
  for (int q = 0; q < 3; ++q) vel[3 * i + q] *= lambda;
}

void launch_leapfrog(const MdArgs& a, cudaStream_t st) {
  if (a.n == 0) return;
  k_leapfrog<<<(a.n + 255) / 256, 256, 0, st>>>(a);
  count_launch();
}

void launch_force_check(const MdArgs& a, cudaStream_t st) {
  if (a.n == 0) return;
  k_force_check<<<(3 * a.n + 255) / 256, 256, 0, st>>>(3 * a.n, a.F, a.err, a.step);
  count_launch();
}

void launch_energy_record(const double* ke_atom, int n, const double* epot, double* rec, long step,
                          cudaStream_t st) {
  k_sum<<<1, 1024, 0, st>>>(ke_atom, n, nullptr, 1, epot, rec, step);
  count_launch();
}

void launch_rescale(int n, double* vel, const double* mass, double* ke_atom, double* ke_sum, double temperature,
                    cudaStream_t st) {
  if (n == 0) return;
  k_kinetic<<<(n + 255) / 256, 256, 0, st>>>(n, vel, mass, ke_atom);
  k_sum<<<1, 1024, 0, st>>>(ke_atom, n, ke_sum, 0, nullptr, nullptr, 0);
  k_rescale<<<(n + 255) / 256, 256, 0, st>>>(n, vel, ke_sum, temperature);
  count_launch();
  count_launch();
  count_launch();
}

}  // namespace nb
