// precision variant: u storage double, u_f storage double, operator MODE_DD
#include "gb_solver.cuh"

const VariantOps* gb_variant_d_d_dd() { return Impl<double, double, MODE_DD>::table(); }
