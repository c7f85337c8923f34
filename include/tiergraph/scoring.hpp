// Forwarder: reference proj/include/tiergraph/scoring.hpp -> the B200 drop-in API.
#pragma once
#include "tiergraph/tiergraph.hpp"
