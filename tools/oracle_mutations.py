# Mutation check of the oracle pins: each plausible mistake must fail a pin test
# (operator, geometry, gather-scatter, Jacobi, PCG incl. the singular
# projections and the weighted stopping norm, GMRES; and the hybrid-Schwarz
# multigrid / FGMRES oracle in oracle/hsmg.py).
# Run from the repo root: python tools/oracle_mutations.py
import subprocess, sys, shutil
src = 'oracle/sem_oracle.c'
orig = open(src).read()
muts = [
 ("qr g12<->g13", "qr[p] = hh * (g11 * ur + g12 * us + g13 * ut);", "qr[p] = hh * (g11 * ur + g13 * us + g12 * ut);"),
 ("R sign", "R[0][1] = (X[0][2] * X[2][1] - X[0][1] * X[2][2]) / J;", "R[0][1] = (X[0][1] * X[2][2] - X[0][2] * X[2][1]) / J;"),
 ("transposed D", "for (int l = 0; l < lx; ++l) s += D[l * lx + j] * qs[IDX(i, l, k)];", "for (int l = 0; l < lx; ++l) s += D[j * lx + l] * qs[IDX(i, l, k)];"),
 ("dssum skip", "  for (int64_t l = 0; l < nloc; ++l) u[l] = v[ids[l]];", "  for (int64_t l = 1; l < nloc; ++l) u[l] = v[ids[l]];"),
 ("jacobi cross", "s += 2.0 * D[i * lx + i] * D[k * lx + k] * H1AT(p) * Ge[4 * n3 + p];", ""),
 ("pcg beta", "const double beta = (k == 1) ? 0.0 : rtz / rtz_prev;", "const double beta = (k == 1) ? 0.0 : rtz_prev / rtz;"),
 ("gll weight", "w[i] = 2.0 / (N * (N + 1.0) * L * L);", "w[i] = 2.0 / (N * (N + 1.0) * L);"),
 ("h2 term", "if (hm != 0.0) s += hm * B[(size_t)e * n3 + p] * ue[p];", "if (hm != 0.0) s += hm * ue[p];"),
 ("weights in G", "G[((size_t)e * 6 + c) * n3 + IDX(i, j, k)] = W * J * s;", "G[((size_t)e * 6 + c) * n3 + IDX(i, j, k)] = J * s;"),
 ("no b projection", "    for (int64_t l = 0; l < n; ++l) r[l] -= mean;", "    (void)mean;"),
 ("no x projection", "    for (int64_t l = 0; l < n; ++l) x[l] -= mean;", "    (void)mean;"),
 ("unweighted stop", "    rn = sqrt(wdot(n, mult, r, r));", "    rn = 0.0; for (int64_t l = 0; l < n; ++l) rn += r[l] * r[l]; rn = sqrt(rn);"),
 ("gmres g sign", "      g[j + 1] = -sn[j] * g[j];", "      g[j + 1] = sn[j] * g[j];"),
 ("gmres rotation", "        H[i * m + j] = cs[i] * a + sn[i] * c;", "        H[i * m + j] = cs[i] * a - sn[i] * c;"),
 ("gmres no precond", "      for (int64_t l = 0; l < n; ++l) z[l] = dinv[l] * vj[l];", "      for (int64_t l = 0; l < n; ++l) z[l] = vj[l];"),
 ("gmres stale restart", "    for (int64_t l = 0; l < n; ++l) r[l] = b[l] - (mask ? mask[l] * w[l] : w[l]);", "    for (int64_t l = 0; l < n; ++l) r[l] = b[l];"),
 ("mask any->all", "if (d) dir[ids[(size_t)e * n3 + IDX(i, j, k)]] = 1;", "if (d && e % 2) dir[ids[(size_t)e * n3 + IDX(i, j, k)]] = 1;"),
]
hsrc = 'oracle/hsmg.py'
horig = open(hsrc).read()
hmuts = [
 ("fdm no nb share", "    Ae[0, 0] += A[N, N]", "    Ae[0, 0] += 0.0"),
 ("fdm lambda scale", "    lam = 4.0 * mu", "    lam = 2.0 * mu"),
 ("fdm volume factor", "out[e] = rh[e] / den * (8.0 / (Lx * Ly * Lz))", "out[e] = rh[e] / den * (1.0 / (Lx * Ly * Lz))"),
 ("fdm Lx<->Lz", "lam[None, None, :] / Lx ** 2", "lam[None, None, :] / Lz ** 2"),
 ("lengths wrong edge", "X[:, :, a, b, N] - X[:, :, a, b, 0]", "X[:, :, a, b, N] - X[:, :, a, 0, b]"),
 ("lagrange sign", "J[:, b] *= (x_to - x_from[q])", "J[:, b] *= (x_to + x_from[q])"),
 ("restrict no 1/m", 'np.asarray(r_f).ravel() * lev_f["mult"]', "np.asarray(r_f).ravel()"),
 ("schwarz no average", 'z = O.dssum(lev["ids"], z, lev["nuniq"]) * lev["mult"]', 'z = O.dssum(lev["ids"], z, lev["nuniq"])'),
 ("vcycle no residual", "        res = rs[l] - level_ax(levels[l], z, h1c, h2c)", "        res = rs[l]"),
 ("vcycle overwrite", "        zs[l] = zs[l] + prolong(levels[l], zs[l + 1])", "        zs[l] = prolong(levels[l], zs[l + 1])"),
 ("fgmres x from V", "            x = x + y[i] * Z[i]", "            x = x + y[i] * V[i]"),
 ("fgmres no b mask", "        b = b * mask", "        b = b"),
]
try:
    for name, a, b in hmuts:
        assert a in horig, name
        open(hsrc, 'w').write(horig.replace(a, b))
        r = subprocess.run([sys.executable, '-m', 'pytest', '-x', '-q', 'tests/test_oracle_hsmg.py', '-p', 'no:cacheprovider'], capture_output=True, text=True)
        print(f"{name:20s} -> {'CAUGHT' if r.returncode else 'MISSED'}  {r.stdout.strip().splitlines()[-1]}", flush=True)
finally:
    open(hsrc, 'w').write(horig)
if '--hsmg-only' in sys.argv:
    sys.exit(0)
try:
    for name, a, b in muts:
        assert a in orig, name
        open(src, 'w').write(orig.replace(a, b))
        r = subprocess.run([sys.executable, '-m', 'pytest', '-x', '-q', 'tests/test_oracle_gll.py', 'tests/test_oracle_operator.py', 'tests/test_oracle_numbering.py', 'tests/test_oracle_pcg.py', 'tests/test_oracle_gmres.py', '-p', 'no:cacheprovider'], capture_output=True, text=True)
        print(f"{name:20s} -> {'CAUGHT' if r.returncode else 'MISSED'}  {r.stdout.strip().splitlines()[-1]}")
finally:
    open(src, 'w').write(orig)
