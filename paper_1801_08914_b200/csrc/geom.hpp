// Mapped-geometry FE path (config 4), see geom.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/hdivred_b200.h"
#include "hdr_device.cuh"
#include "hdr_internal.hpp"

namespace hdr {

struct GeomState;
GeomState* geom_create(const RefElement& re, const DevMesh& dm, const std::vector<int>& mbase, const double h[3],
                       int64_t m, int64_t ndofs, const double* verts_host, bool weighted, cudaStream_t st);
bool geom_mapped(const GeomState* G);
void geom_destroy(GeomState* G);
int64_t geom_nnz_h(const GeomState* G);
hdr_status geom_hybridize(GeomState* G, const double* alpha, const double* beta, const double* f, double* hval,
                          double* g, cudaStream_t st);
hdr_status geom_recover_hybrid(GeomState* G, const double* alpha, const double* beta, const double* lambda,
                               const double* f, double* x_hat, double* x, cudaStream_t st);
hdr_status geom_condense(GeomState* G, const double* alpha, const double* beta, const double* f, double* sval,
                         double* fs, cudaStream_t st);
hdr_status geom_recover_condensed(GeomState* G, const double* alpha, const double* beta, const double* x_b,
                                  const double* f, double* x, cudaStream_t st);
const double* geom_element_blocks(const GeomState* G);
// A_T of every cell (mapped: Piola assembly; affine weighted: fl(fl(alpha D) + fl(beta M)))
void geom_assemble_blocks(GeomState* G, const double* alpha, const double* beta, cudaStream_t st);

}  // namespace hdr
