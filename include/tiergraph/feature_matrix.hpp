// Forwarder: reference proj/include/tiergraph/feature_matrix.hpp -> the B200 drop-in API.
#pragma once
#include "tiergraph/tiergraph.hpp"
