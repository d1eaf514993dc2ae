"""Application drivers of the paper's Section 6, SURVEY NEXT #4.

Each driver builds its linear system on the host (seeded, synthetic), solves it
with the GPU library (`paper_2509_19267_b200.Solver`, the same C ABI as the
bench) and reports the application's own metric:

* `fem_poisson`  — P1 FEM Poisson on the unit square, relative L2
  error of the nodal solution against sin(pi x) sin(pi y) (tab:poisson_helmholtz).
* `deblur`       — 3-channel image deblurring with the banded Gaussian Toeplitz
  operator eq:toeplitz, PSNR / SSIM per channel (tab:image).
* `pps_filter`   — denoising filter for the predator-prey-scavenger model
  (P:827-916): M_v c_v = v from noisy delayed populations, prediction error.

None of this is on the hot path; the drivers only call the library.
"""
