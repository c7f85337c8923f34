// Forwarder: reference proj/include/tiergraph/sampling.hpp -> the B200 drop-in API.
#pragma once
#include "tiergraph/tiergraph.hpp"
