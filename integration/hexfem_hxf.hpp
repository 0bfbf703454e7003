// Reference-side integration of the B200 backend: the hexfem hot-path API
// (proj/include/hexfem/operator.hpp:53-64, restriction.hpp:33-50,
// contraction.hpp:43-75, tensor_basis.hpp:38-47, bench.hpp:71-72,95)
// re-implemented over the hxf C-ABI (include/hxf.h), signature for signature,
// so existing hexfem callers switch by namespace (or by linking this file in
// place of the reference's definitions).  Compiled against the reference's
// own headers.
#pragma once

#include <array>
#include <cstdint>
#include <span>
#include <vector>

#include "hexfem/bench.hpp"
#include "hexfem/contraction.hpp"
#include "hexfem/operator.hpp"
#include "hexfem/restriction.hpp"
#include "hexfem/tensor_basis.hpp"

namespace hexfem::hxf_backend {

// operator.hpp:56-58 — y = (alpha A + beta B) x on the GPU (host spans: H2D,
// kernel, D2H).  pool / scratch accepted and ignored (the GPU is the worker).
// op.plan.flops (if set) is credited with the sum-factorized count the
// reference's instrumented kernels would record (2 chains per component and
// stage, flops_estimate per element).
void operator_apply(const MatFreeOperator& op, std::span<const double> x, std::span<double> y,
                    ThreadPool* pool = nullptr, OperatorScratch* scratch = nullptr);

// operator.hpp:63-64
std::vector<double> operator_diagonal(const MatFreeOperator& op, ThreadPool* pool = nullptr);

// pcg.hpp:38-41 specialised to the operator: device-resident PCG, only b in
// and x + the report out (the signature-compatible ApplyFn route would pay
// H2D + D2H per apply).
SolveReport pcg(const MatFreeOperator& op, std::span<const double> b,
                std::span<const double> jacobi_diag, const PcgOptions& options, std::span<double> x);

// bench.hpp:71-72 / bench.cpp:121-137
BpSolveResult solve_bp(const BpProblem& problem, ThreadPool* pool = nullptr, bool jacobi = true);

// restriction.hpp:35-50 — on the GPU; G^T in the reference's colour order
// (bitwise equal) for the structured box make_restriction builds.
void apply_g(const ElemRestriction& r, std::span<const double> l_vec, std::span<double> e_vec,
             ThreadPool* pool = nullptr);
void apply_g_transpose(const ElemRestriction& r, std::span<const double> e_vec,
                       std::span<double> l_vec, ThreadPool* pool = nullptr);
std::vector<double> multiplicity(const ElemRestriction& r);
void gather_scalar(const ElemRestriction& r, std::span<const double> e_scalar,
                   std::span<double> l_scalar, ThreadPool* pool = nullptr);

// contraction.hpp:51-75 — the sum-factorized path on the GPU (plan.path is
// ignored: KernelPath::Naive is the reference's oracle path); plan.flops is
// credited exactly as the reference's FlopCounter would be.
void contract_batch(const KernelPlan& plan, std::span<const double> matrix, int n_out, int n_in,
                    int dim, std::array<int, 3> in_shape, std::int64_t ne,
                    std::span<const double> in, std::span<double> out, bool accumulate = false);
void apply_basis_batch(const KernelPlan& plan, const TensorBasis& basis, EvalMode mode,
                       EvalDirection dir, std::int64_t ne, std::span<const double> in,
                       std::span<double> out, ContractionScratch& scratch);
std::uint64_t flops_estimate(const KernelPlan& plan, EvalMode mode);

// tensor_basis.hpp:46-47
void apply_tensor_3d(const TensorBasis& basis, EvalMode mode, EvalDirection dir, int m,
                     std::span<const double> u, std::span<double> v);

// Drop the cached device copy of one operator / every cached device object.
void release(const MatFreeOperator& op);
void release_all();

}  // namespace hexfem::hxf_backend
