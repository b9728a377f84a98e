// precision variant: u storage float, u_f storage float, operator MODE_F32
#include "gb_solver.cuh"

const VariantOps* gb_variant_f_f_f32() { return Impl<float, float, MODE_F32>::table(); }
