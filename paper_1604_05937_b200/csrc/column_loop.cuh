// Device helpers shared by the column-loop kernels.
#pragma once

namespace pm {

// |det J| of the affine map reference prism -> physical prism cell-layer.
// Vertex index v = 2a + b (a: triangle vertex, b: 0 bottom / 1 top level).
// Same operation order as the oracle (oracle/prismesh_oracle.c).
__device__ __forceinline__ double prism_abs_detj(const double *X,
                                                 const double *Y,
                                                 const double *Z) {
  const double xm0 = 0.5 * (X[0] + X[1]), ym0 = 0.5 * (Y[0] + Y[1]);
  const double xm1 = 0.5 * (X[2] + X[3]), ym1 = 0.5 * (Y[2] + Y[3]);
  const double xm2 = 0.5 * (X[4] + X[5]), ym2 = 0.5 * (Y[4] + Y[5]);
  const double a2 = (xm1 - xm0) * (ym2 - ym0) - (xm2 - xm0) * (ym1 - ym0);
  const double h = ((Z[1] - Z[0]) + (Z[3] - Z[2]) + (Z[5] - Z[4])) / 3.0;
  return fabs(a2 * h);
}

} // namespace pm
