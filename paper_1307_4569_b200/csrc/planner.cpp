// planner.cpp -- host-side lattice planning for the shear algorithm.
//
//  * normal form: b = L/M, N = L/a, s = b*lambda1/lambda2
//  * feasibility: L a multiple of L_min = lambda2*lcm(a,M) (Prop. minsig)
//  * shear: U^{-1}_{s0,s1} A = D V with X = gcd(s1 a + s, b), Bezout X = k1(s1 a+s) + k2 b
//    and Eq. (modcond) mod(s0 X + a k1, ab/X) = 0.  We enumerate s1
//    and SOLVE (modcond) for s0 (any solution is valid -- reading Z9 of DESIGN.md).
//    The time-only shear (s0 = 0) exists iff (s1 a + s) = 0 mod b is solvable.
//  * b_r = X (reading Z6), a_r = ab/b_r, M_r = L/b_r, N_r = L/a_r (Alg. 1 line 17).
//  * inner separable lattice (c,d,p,q) by Eqs. (cd),(pq).
//  * Alg. 1 constants C1..C6, reduced mod 2N (C6 mod L).
#include "planner.hpp"

#include <cstdio>
#include <vector>

namespace nsdgt {

int64_t gcd64(int64_t x, int64_t y) {
    if (x < 0) x = -x;
    if (y < 0) y = -y;
    while (y) {
        int64_t t = x % y;
        x = y;
        y = t;
    }
    return x;
}

int64_t lcm64(int64_t x, int64_t y) { return x / gcd64(x, y) * y; }

int64_t mod64(int64_t x, int64_t m) {
    int64_t r = x % m;
    return r < 0 ? r + m : r;
}

int64_t mulmod64(int64_t x, int64_t y, int64_t m) {
    return (int64_t)((__int128)mod64(x, m) * (__int128)mod64(y, m) % (__int128)m);
}

void egcd64(int64_t x, int64_t y, int64_t* X, int64_t* k1, int64_t* k2) {
    // iterative extended Euclid on (x, y)
    int64_t r0 = x, r1 = y, s0 = 1, s1 = 0, t0 = 0, t1 = 1;
    while (r1 != 0) {
        int64_t qq = r0 / r1;
        int64_t tmp = r0 - qq * r1; r0 = r1; r1 = tmp;
        tmp = s0 - qq * s1; s0 = s1; s1 = tmp;
        tmp = t0 - qq * t1; t0 = t1; t1 = tmp;
    }
    if (r0 < 0) { r0 = -r0; s0 = -s0; t0 = -t0; }
    *X = r0; *k1 = s0; *k2 = t0;
}

static int64_t modinv64(int64_t x, int64_t m) {
    if (m == 1) return 0;
    int64_t g, k1, k2;
    egcd64(mod64(x, m), m, &g, &k1, &k2);
    return g == 1 ? mod64(k1, m) : -1;
}

namespace {

struct Cand {
    int64_t s0, s1, X;
};

// Solve Eq. (modcond) for s0 given s1.  Returns false if no s0 exists.
bool solve_s0(int64_t a, int64_t b, int64_t s, int64_t L, int64_t s1, Cand* c) {
    int64_t X, k1, k2;
    egcd64(s1 * a + s, b, &X, &k1, &k2);
    if (X == 0) return false;
    const int64_t Mo = a * b / X;
    const int64_t gp = gcd64(X, Mo);
    if (mod64(a * k1, gp) != 0) return false;
    const int64_t m = Mo / gp;
    int64_t s0 = 0;
    if (m > 1) {
        const int64_t inv = modinv64(X / gp, m);
        if (inv < 0) return false;
        const int64_t t = (a * k1) / gp;
        s0 = mulmod64(-t, inv, m);
    }
    // verify (modcond) exactly
    if (mod64((__int128)s0 * X % Mo + (__int128)a * k1 % Mo, Mo) != 0) {
        // fall back to a direct search over one period (tiny m only)
        bool ok = false;
        for (int64_t t = 0; t < m && t < 1000000; ++t)
            if (mod64((__int128)t * X % Mo + (__int128)a * k1 % Mo, Mo) == 0) { s0 = t; ok = true; break; }
        if (!ok) return false;
    }
    (void)L;
    c->s0 = s0;
    c->s1 = s1;
    c->X = X;
    return true;
}

void inner_shape(dgt_lattice_info* o) {
    o->c = gcd64(o->ia, o->iM);
    o->d = gcd64(o->ib, o->iN);
    o->p = o->ia / o->c;
    o->q = o->iM / o->c;
}

int64_t prime_exponent(int64_t x, int64_t p) {
    if (x == 0) return 64;
    int64_t e = 0;
    while (x % p == 0) { x /= p; ++e; }
    return e;
}

// Eq. (s1choice): s1 = prod p_j^{mu_j}, mu_j = 1 iff alpha_j = sigma_j,
// over the primes p_j of L (alpha_j, sigma_j the exponents of p_j in a and s).
int64_t paper_s1(int64_t L, int64_t a, int64_t s) {
    int64_t s1 = 1, x = L;
    for (int64_t p = 2; p * p <= x || x > 1; ++p) {
        if (p * p > x) p = x;  // remaining prime factor
        if (x % p) continue;
        while (x % p == 0) x /= p;
        if (prime_exponent(a, p) == prime_exponent(s, p)) s1 *= p;
        if (x == 1) break;
    }
    return s1;
}

}  // namespace

int plan_lattice(int64_t L, int64_t a, int64_t M, int64_t lam1, int64_t lam2, int flags,
                 bool force, int64_t s0_in, int64_t s1_in, dgt_lattice_info* o, std::string* err) {
    char buf[256];
    if (!o) { *err = "null output"; return DGT_EINVAL; }
    *o = dgt_lattice_info{};
    if (L <= 0 || a <= 0 || M <= 0) { *err = "L, a, M must be positive"; return DGT_EINVAL; }
    if (lam2 < 1 || lam1 < 0 || lam1 >= lam2) { *err = "need 0 <= lambda1 < lambda2"; return DGT_EINVAL; }
    if (gcd64(lam1, lam2) != 1) { *err = "gcd(lambda1, lambda2) must be 1"; return DGT_EINVAL; }
    o->L = L; o->a = a; o->M = M; o->lambda1 = lam1; o->lambda2 = lam2;
    o->L_min = lam2 * lcm64(a, M);
    if (L % a || L % M || L % o->L_min) {
        std::snprintf(buf, sizeof buf, "illegal transform length L=%lld; L must be a multiple of L_min=%lld",
                      (long long)L, (long long)o->L_min);
        *err = buf;
        return DGT_EILLEGAL_LENGTH;
    }
    const int64_t b = L / M, N = L / a, s = b * lam1 / lam2;
    o->b = b; o->N = N; o->s = s;
    const int64_t twoN = 2 * N;

    Cand ch{0, 0, b};
    if (force) {
        ch.s1 = mod64(s1_in, b > 0 ? L : 1);
        if (!solve_s0(a, b, s, L, mod64(ch.s1, b), &ch)) { *err = "forced s1 admits no s0"; return DGT_EINVAL; }
        ch.s1 = mod64(s1_in, L);
        // validate the given s0 against (modcond)
        int64_t X, k1, k2;
        egcd64(ch.s1 * a % (a * b) + s, b, &X, &k1, &k2);
        const int64_t Mo = a * b / X;
        if (mod64((__int128)mod64(s0_in, L) * X % Mo + (__int128)a * k1 % Mo, Mo) != 0) {
            *err = "forced (s0, s1) violates Eq. (modcond)";
            return DGT_EINVAL;
        }
        ch.s0 = mod64(s0_in, L);
        ch.X = X;
        if (ch.s0 == 0 && X != b) { *err = "s0 = 0 requires s1 a + s = 0 mod b"; return DGT_EINVAL; }
    } else if (s == 0) {
        ch = Cand{0, 0, b};
    } else if (flags & DGT_SHEAR_PAPER) {
        int64_t s1 = paper_s1(L, a, s);
        if (!solve_s0(a, b, s, L, s1, &ch)) { *err = "paper's s1 choice admits no s0"; return DGT_EINVAL; }
        if (ch.X == b) ch.s0 = 0;
    } else {
        // Policy: time-only shear if it exists (no length-L FFT), else the
        // frequency shear with s1 = 0 (no pre-chirp) if valid and small, else least cost.
        bool found = false;
        for (int64_t s1 = 1; s1 < b; ++s1)
            if (mod64(s1 * a + s, b) == 0) { ch = Cand{0, s1, b}; found = true; break; }
        if (!found) {
            int64_t best_cost = INT64_MAX;
            for (int64_t s1 = 0; s1 < b; ++s1) {
                Cand c;
                if (!solve_s0(a, b, s, L, s1, &c)) continue;
                if (c.X == b) continue;  // would be a time shear
                const int64_t ar = a * b / c.X, iM = L / ar, iN = L / c.X;
                const int64_t d = gcd64(ar, iN);
                int64_t cost = d + iM + (s1 != 0 ? 1 : 0);
                if (d > 16384 || iM > 16384) cost += (int64_t)1 << 40;
                if (s1 == 0 && cost < ((int64_t)1 << 40)) { ch = c; found = true; break; }
                if (cost < best_cost) { best_cost = cost; ch = c; found = true; }
            }
            if (!found) { *err = "no valid shear found"; return DGT_EINVAL; }
        }
    }

    o->s0 = ch.s0;
    o->s1 = ch.s1;
    if (s == 0 && ch.s0 == 0 && ch.s1 == 0) o->branch = DGT_BRANCH_SEPARABLE;
    else o->branch = ch.s0 == 0 ? DGT_BRANCH_TIME : DGT_BRANCH_FREQ;

    if (o->branch != DGT_BRANCH_FREQ) {
        o->b_r = b; o->a_r = a; o->M_r = M; o->N_r = N;
        o->ia = a; o->iM = M; o->iN = N; o->ib = b;
        // Alg. 1 line 8: C1 = s1 a (L+1) mod 2N
        o->C1 = mulmod64(mulmod64(o->s1, a, twoN), L + 1, twoN);
        o->chirp_sigma = o->s1;
        o->pre_sigma = 0;
    } else {
        const int64_t br = ch.X, ar = a * b / br;
        o->b_r = br; o->a_r = ar; o->M_r = L / br; o->N_r = L / ar;
        o->ia = br; o->iM = o->N_r; o->iN = o->M_r; o->ib = ar;
        // Alg. 1 lines 17-20
        if (ar % a) { *err = "a_r/a not integral"; return DGT_EINVAL; }
        o->C1 = mod64(ar / a, twoN);
        const __int128 s0br = (__int128)ch.s0 * br;
        if (s0br % a) { *err = "C2 = -s0 b_r / a not integral (reading Z8)"; return DGT_EINVAL; }
        const int64_t C2 = mod64((int64_t)(-(s0br / a) % twoN), twoN);
        o->C2 = C2;
        o->C3 = mulmod64(mulmod64(a, o->s1, twoN), L + 1, twoN);
        o->C4 = mulmod64(mulmod64(C2, br, twoN), L + 1, twoN);
        o->C5 = mulmod64(2 * o->C1, br, twoN);
        o->C6 = mulmod64(mulmod64(ch.s0, o->s1, L) + 1, br, L);
        o->chirp_sigma = mod64(-ch.s0, 2 * L);
        o->pre_sigma = o->s1;
    }
    inner_shape(o);
    return DGT_OK;
}

}  // namespace nsdgt
