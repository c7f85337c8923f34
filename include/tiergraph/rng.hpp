// Forwarder: reference proj/include/tiergraph/rng.hpp -> the B200 drop-in API.
#pragma once
#include "tiergraph/tiergraph.hpp"
