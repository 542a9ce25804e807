// semikern_b200/semikern.hpp -- header-only C++ shim that re-exposes the
// reference library's API (namespace semikern, proj/include/semikern/
// {error,rng,semiring,matrix,matgen,matio,dnn,bench}.hpp) on top of the C-ABI
// in sk_api.h, so reference code compiles against the B200 engine unchanged.
// The per-header files live in include/semikern_b200/semikern/ under the
// reference's own names: put `-I include/semikern_b200 -I include` where the
// reference's include directory was, and `#include "semikern/dnn.hpp"` resolves
// here.  tests/cpp/Makefile compiles the reference's own acceptance suite
// (proj/tests/acceptance.cpp) that way, untouched.
//
//   #include "semikern/dnn.hpp"          // or "semikern_b200/semikern.hpp"
//   using namespace semikern;
//   CsrMatrix w = csr_from_triples(m, m, triples);
//   Batch y = relu_forward(DnnModel({Matrix(w)}, {bias}), input);
//
// Differences a caller can observe, all deliberate:
//  * Matrices live in device memory.  Element access goes through a host mirror
//    (DenseMatrix: read-write, uploaded again before the next kernel reads it;
//    CsrMatrix: immutable views of a host copy fetched once).
//  * Copies share storage until written (copy on write), so value semantics hold.
//  * `workers` is accepted and checked (>= 1); results are bitwise independent
//    of it, as the reference guarantees (dnn.hpp:75-76).
//  * ForwardOptions gains `clip` (BASELINE cfg3-5); relu_forward_sparse() and
//    categories() are extensions for the sparse-activation workloads.
//  * Device allocation failure raises OutOfMemory (a semikern::Error).
#pragma once

#include "semikern/error.hpp"
#include "semikern/rng.hpp"
#include "semikern/semiring.hpp"
#include "semikern/matrix.hpp"
#include "semikern/matgen.hpp"
#include "semikern/matio.hpp"
#include "semikern/dnn.hpp"
#include "semikern/bench.hpp"
