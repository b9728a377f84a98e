// precision variant: u storage double, u_f storage __half, operator MODE_DD
#include "gb_solver.cuh"

const VariantOps* gb_variant_d_h_dd() { return Impl<double, __half, MODE_DD>::table(); }
