// hiercva_gpu.hpp -- the maintainer-side binding of libhcva_gpu.so into the
// reference library (hiercva, /root/reference/proj): drop-ins with the
// reference's own signatures and types for the hot-path functions, over the
// C ABI of include/hcva_gpu.h.  Compiled against proj/include; only the
// headers that do not need Eigen (market / defaults / portfolio / rng /
// errors) are included, so this builds wherever the reference core builds.
#pragma once

#include <cstdint>
#include <vector>

#include "hiercva/defaults.hpp"
#include "hiercva/market.hpp"
#include "hiercva/portfolio.hpp"
#include "hiercva/rng.hpp"

namespace hiercva::gpu {

// The three blocks of hiercva::SimulationSet (pipeline.hpp:19-23), in the
// same order; a build with pipeline.hpp returns SimulationSet{std::move(...)}.
struct SimulationBlocks {
    MarketBlock market;
    DefaultBlock defaults;
    MtMCube cube;
};

// The Philox key of a RandomStream (rng.cpp:44-55): root key of its seed,
// split along its lineage.
std::uint64_t stream_key(const RandomStream& stream);

// simulate_set (pipeline.cpp:63-70): market from stream.split(0)
// (simulate_market, market.cpp:161-234), defaults from stream.split(1)
// (sample_default_block, defaults.cpp:20-45), cube (build_mtm_cube,
// portfolio.cpp:97-147) -- on the GPU, exported into the reference's blocks.
// Errors are the reference's exception types (errors.hpp:9-25).
SimulationBlocks simulate_set_gpu(const ModelParams& params, const TimeGrid& grid,
                                  const std::vector<SwapSpec>& book, int n_paths, int n_replicas,
                                  const RandomStream& stream);

// simulate_market (market.hpp:144-145) alone.
MarketBlock simulate_market_gpu(const ModelParams& params, const TimeGrid& grid, int n_paths,
                                const RandomStream& stream);

}  // namespace hiercva::gpu
