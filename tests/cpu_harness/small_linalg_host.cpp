// Host (g++) instantiation of the device small-linear-algebra routines, so
// tests/test_small_linalg_cpu.py can check the exact kernel code against
// numpy on a machine without a GPU.  Test infrastructure only.
#include <cstring>
#include <vector>

#include "../../paper_1807_01350_b200/csrc/small_linalg.cuh"

using namespace octen;

extern "C" {

void h_jacobi_eig(int n, const double* a, double* w, double* v) {
    std::vector<double> am(a, a + (size_t)n * n), cs(2 * (n + 2));
    std::vector<int> iw(n + 8);
    TeamHost team;
    jacobi_eig_sym(team, n, am.data(), v, cs.data(), iw.data());
    for (int i = 0; i < n; ++i) w[i] = am[i + (size_t)n * i];
}

int h_eig_real(int n, const double* a, double* wr, double* wi, double* v) {
    std::vector<double> h(a, a + (size_t)n * n), ort(n);
    return eig_real(n, h.data(), v, wr, wi, ort.data()) ? 1 : 0;
}

int h_lu_inverse(int n, const double* a, double* inv) {
    std::vector<double> m(a, a + (size_t)n * n);
    std::vector<int> rp(n), cp(n);
    return lu_fullpiv_inverse(n, m.data(), n, inv, n, rp.data(), cp.data()) ? 1 : 0;
}

int h_chol_semidef(int n, double* a, double tol) { return chol_semidef(n, a, n, tol); }

int h_greedy(int r, const double* sim, double tie, int* perm) {
    std::vector<unsigned char> a(r), b(r);
    return greedy_match(r, sim, r, tie, perm, a.data(), b.data());
}

double h_top_sv(int m, int n, const double* a, double* u, double* v) {
    std::vector<double> red(1 + 2 + n + 8);
    TeamHost team;
    return top_singular_pair(team, m, n, a, u, v, red.data());
}

void h_mt64(unsigned long long seed, int n, double* out) {
    Mt64 g;
    g.seed(seed);
    for (int i = 0; i < n; ++i) out[i] = g.uniform01();
}

}  // extern "C"

extern "C" int h_team_chol_inv(int n, double* a, double* inv, double tol) {
    TeamHost team;
    double sc[2];
    int ir[2];
    const int rk = team_chol_semidef(team, n, a, n, tol, sc, ir);
    team_tri_inv_lower(team, n, a, n, inv, n);
    return rk;
}

extern "C" int h_subspace_eig_top(int n, const double* a, int k, int m, double* u, double* theta) {
    std::vector<double> w((size_t)n * m), h((size_t)m * m), hv((size_t)m * m), cs(2 * (m + 2) + 1 + 2);
    std::vector<double> ub((size_t)n * m);
    std::vector<int> iw(2 * m + 8);
    TeamHost team;
    const int ok = subspace_eig_top(team, n, a, k, m, ub.data(), w.data(), h.data(), hv.data(), theta,
                                    cs.data(), iw.data());
    for (size_t e = 0; e < (size_t)n * k; ++e) u[e] = ub[e];
    return ok;
}

extern "C" int h_eig_real_team(int n, const double* a, double* wr, double* wi, double* v) {
    std::vector<double> h(a, a + (size_t)n * n), ort(n);
    TeamHost team;
    return eig_real_team(team, n, h.data(), v, wr, wi, ort.data()) ? 1 : 0;
}

extern "C" int h_lu_inverse_team(int n, const double* a, double* inv) {
    std::vector<double> m(a, a + (size_t)n * n), piv(n), scr(4);
    std::vector<int> rp(n), cp(n);
    TeamHost team;
    return lu_fullpiv_inverse_team(team, n, m.data(), n, inv, n, rp.data(), cp.data(), piv.data(), scr.data()) ? 1
                                                                                                             : 0;
}

extern "C" int h_sym_eig_top_tridiag(int n, const double* a, int k, double* u, double* theta, int kb) {
    std::vector<double> am(a, a + (size_t)n * n), work((size_t)3 * n + (size_t)5 * n * kb), cf(k + 8), red(8);
    TeamHost team;
    return sym_eig_top_tridiag(team, n, am.data(), k, u, theta, work.data(), kb, cf.data(), red.data());
}
