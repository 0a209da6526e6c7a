// Chained in-plane FFT passes (axis 1 <-> axis 2) through an L2-resident
// scratch ring, in ONE persistent kernel.
//
// The axis-1 and axis-2 transforms of a z-plane depend only on that plane, so
// for a chunk of G planes the second pass can start as soon as the first has
// written the chunk.  Work items (A tiles of chunk c, then B tiles of chunk c)
// are dequeued in the order A0 A1 B0 A2 B1 ... from a global counter; a B tile
// spins until all A tiles of its chunk are done, and an A tile waits until the
// ring slot it overwrites has been drained.  Every wait points at an item that
// was dequeued earlier by a resident CTA, so the schedule cannot deadlock.
// HBM sees the first pass's input and the second pass's output only: the
// intermediate lives in a ring of R chunks (a few MB) that stays in L2.
//
//   inverse (Tikhonov / TV x-update): A = axis-2 inverse of W -> ring,
//            B = axis-1 inverse c2r of ring -> x (real) + residue reduction
//   forward (TV theta):               A = axis-1 r2c of theta -> ring,
//            B = axis-2 forward of ring -> W
#pragma once

#include "fft.cuh"

namespace vsr {

struct ChainPlan {
    bool ok = false;
    int g = 0;             // planes per chunk
    int chunks = 0;
    int ring = 0;          // slots
    int lookahead = 0;     // chunks of A tiles queued ahead of the B tiles
    size_t a_tiles = 0, b_tiles = 0;  // per chunk
    size_t blocks = 0;     // persistent grid
    size_t scratch_elems = 0;
    size_t b_total() const { return b_tiles * (size_t)chunks; }
};

ChainPlan chain_plan(const Dims& d);

// Device workspace for one chain: scratch ring (complex), queue + done counters.
struct ChainWork {
    double2* ring = nullptr;
    int* counters = nullptr;  // [1 + 2 * chunks]
};

// Inverse: W (complex, axis 3 already inverted) -> axes 2, 1 -> out (real),
// scaled by `scale`; residue partials (2 doubles per B tile, fixed slots) and
// non-finite index as in FftEngine::inverse3 with OUT_REAL.
void launch_chain_inverse(const Dims& d, const ChainPlan& p, const ChainWork& w, const double2* W,
                          double* out, double scale, const PassReduce& red, cudaStream_t st);
// Forward: theta (real) -> axes 1, 2 -> W (complex, unscaled).
void launch_chain_forward(const Dims& d, const ChainPlan& p, const ChainWork& w, const double* theta,
                          double2* W, cudaStream_t st);

}  // namespace vsr
