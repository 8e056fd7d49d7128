// Compile check (g++ -fsyntax-only, tests/test_capi.py): the C++ drop-in shim works with
// the reference's own types.  A reference caller switches by namespace.
#include "sphere/convolution.hpp"
#include "sphere/grid.hpp"
#include "sphere/harmonics.hpp"
#include "sphere_gpu.hpp"

int main() {
    const sphere::GridSpec g = sphere::build_gaussian(16, 32);
    sphere::SphericalField f(g, 2);
    const sphere::SpectralCoeffs c = sphere_gpu::sht_forward(f, 16, 16);
    const sphere::SphericalField r = sphere_gpu::sht_inverse(c, g);
    const sphere_gpu::DiscoOperator op =
        sphere_gpu::assemble_disco(g, sphere::build_gaussian(8, 16), sphere::morlet_basis(1.0));
    sphere::MixTensor mix(3, 2, op.n_basis);
    const sphere::SphericalField y = sphere_gpu::disco_apply(op, r, mix);
    const sphere::SphericalField yt = sphere_gpu::disco_transpose_apply(op, y, mix);
    sphere::SpectralKernel k(2, 2, 16);
    const sphere::SphericalField z = sphere_gpu::spectral_conv(f, k);
    return static_cast<int>(y.data.size() + z.data.size() > 0 ? 0 : 1);
}
