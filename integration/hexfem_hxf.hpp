// Reference-side integration of the B200 backend: the hexfem hot-path API
// (proj/include/hexfem/operator.hpp:53-64, bench.hpp:71-72,95) re-implemented
// over the hxf C-ABI (include/hxf.h), signature for signature, so existing
// hexfem callers switch by namespace (or by linking this file in place of
// operator_apply's definition).  Compiled against the reference's own headers.
#pragma once

#include <span>
#include <vector>

#include "hexfem/bench.hpp"
#include "hexfem/operator.hpp"

namespace hexfem::hxf_backend {

// operator.hpp:56-58 — y = (alpha A + beta B) x on the GPU (host spans: H2D,
// kernel, D2H).  pool / scratch accepted and ignored (the GPU is the worker).
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

// Drop every cached device operator (the side table keyed on the host operator).
void release_all();

}  // namespace hexfem::hxf_backend
