"""Mutation check of the CPU oracle's pins (test infrastructure; not run by pytest).

Each entry is a plausible mistake in `oracle/ctf_oracle.c` (a dropped term, a wrong sign,
index or comparison, a transposed operand).  For each, the script copies oracle/, synthetic/
and tests/ to /tmp, applies the mutation, rebuilds the oracle and runs the CPU pins
(tests/test_oracle_pins.py, tests/test_oracle_bicubic.py).  KILLED = some pin fails.
Expected survivors are listed in DESIGN.md §3 with the reason (equivalent mutants, or
conventions the paper leaves free).   Usage: python scripts/oracle_mutants.py [name ...]
"""
import subprocess, shutil, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MUTS = {
 'f_weights_swap': ("L->w[1] = s * (1.0 - t);\n    L->w[2] = (1.0 - s) * t;", "L->w[1] = (1.0 - s) * t;\n    L->w[2] = s * (1.0 - t);"),
 'g_eq1_Nplus1': ("else c[ch] = Swp[ch] + (1.0 - Sw) * Sp[ch] / N;", "else c[ch] = Swp[ch] + (1.0 - Sw) * Sp[ch] / (N + 1);"),
 'h_zero_weight_known': ("if (dw[j] == 0.0) continue;               /* only", "if (0) continue;               /* only"),
 'j_eq2_half_down': ("long num = 2L * (a - 1) * (c - n) + (a - 1 - n);", "long num = 2L * (a - 1) * (c - n) + (a - 1 - n) - 1;"),
 'k_mag_strict': ("L->magnified = (r2 <= 1.0f);", "L->magnified = (r2 < 1.0f);"),
 'm_mask16_15': ("ok = bw <= 16 && bh <= 16 && n <= a;", "ok = bw <= 15 && bh <= 15 && n <= a;"),
 'n_cplus_extra_pick_ge': ("if (cum > target) { pick = q; break; }\n            }\n            prod[c]", "if (cum >= target) { pick = q; break; }\n            }\n            prod[c]"),
 'o_stf_le': ("int dx = u[0] < (double)L->s;", "int dx = u[0] <= (double)L->s;"),
 'p_stf_swap_uv': ("int dx = u[0] < (double)L->s;\n    int dy = u[1] < (double)L->t;", "int dx = u[1] < (double)L->s;\n    int dy = u[0] < (double)L->t;"),
 'q_cplus_candidates_from_c': ("const lane_t *Ll = &L[l];", "const lane_t *Ll = &L[c];"),
 'r_wc_Sw_plus': ("if (wc) c[ch] = Swp[ch] / Sw;", "if (wc) c[ch] = Swp[ch];"),
 's_eq1_no_allknown': ("if (all_known) { blend_exact(tex, L, c); return; }       /* P:482-483 */", ""),
 't_eq1_no_N1': ("if (N == 1) { for (int ch = 0; ch < 4; ++ch) c[ch] = plast[ch]; return; }  /* P:479-481 */", ""),
 'u_list_n_lt_a': ("else ok = n <= a;                                                     /* List, R-6 */", "else ok = n < a;"),
 'v_producer_identity': ("for (int r = 0; r < n; ++r) prod[act[r]] = U[r];", "for (int r = 0; r < n; ++r) prod[r] = U[r];"),
 'w_box_transposed': ("prod[act[i]] = (uint32_t)(miny + i / bw) * (uint32_t)tex->W + (uint32_t)(minx + i % bw);", "prod[act[i]] = (uint32_t)(miny + i % bh) * (uint32_t)tex->W + (uint32_t)(minx + i / bh);"),
 'x_philox_key': ("if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }", "if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE84u; }"),
 'y_evals_cplus': ("        evals = nprod;\n    }\n\n    if (a == 0)", "        evals = np;\n    }\n\n    if (a == 0)"),
 'z_magnified_any': ("if (L[lane].active && !L[lane].magnified) magnified = 0;\n    }\n\n    /* lanes", "if (L[lane].active && L[lane].magnified) magnified = 1;\n    }\n\n    /* lanes"),
 'aa_bc1_3mode_alpha': ("out[3] = (c0 > c1 || code != 3) ? 255 : 0;", "out[3] = (c0 >= c1 || code != 3) ? 255 : 0;"),
 'ab_footprint_floor_trunc': ("float flx = floorf(fx), fly = floorf(fy);\n    int x0 = (int)flx, y0 = (int)fly;\n    st[0]", "float flx = truncf(fx), fly = truncf(fy);\n    int x0 = (int)flx, y0 = (int)fly;\n    st[0]"),
 # the three mutants of the round-1 verdict
 'v1a_eq1_as_wc': ("if (wc) c[ch] = Swp[ch] / Sw;", "if (1) c[ch] = Swp[ch] / Sw;"),
 'v1b_jacobian_transposed': ("float rx = a0 + a1, ry = a2 + a3;\n        float r2", "float rx = a0 + a2, ry = a1 + a3;\n        float r2"),
 'v1c_eq2_ignores_a': ("long num = 2L * (a - 1) * (c - n) + (a - 1 - n);\n    long den = 2L * (a - 1 - n);", "long num = 2L * (31) * (c - n) + (31 - n);\n    long den = 2L * (31 - n);"),
 # bicubic (R-24 .. R-28)
 'bb_bspline_w1_sign': ("w[1] = ((3.0f * s3 - 6.0f * s2) + 4.0f) / 6.0f;", "w[1] = ((3.0f * s3 + 6.0f * s2) + 4.0f) / 6.0f;"),
 'bc_cr_w0_w3_swap': ("w[0] = -0.5f * (s * r2);", "w[0] = -0.5f * (s2 * r);"),
 'bd_cubic_pick_signed': ("for (int i = 0; i < 4; ++i) { S = S + fabsf(w[i]); if (w[i] != 0.0f) last = i; }", "for (int i = 0; i < 4; ++i) { S = S + w[i]; if (w[i] != 0.0f) last = i; }"),
 'be_positivized_neg_sign': ("c[ch] += (lobe ? -(double)Wl : (double)Wl) * p[ch];", "c[ch] += (double)Wl * p[ch];"),
 'bf_bicubic_cap_ignores_E': ("const int cap = E * a;", "const int cap = a;"),
 'bg_tap_offset': ("L->x[i] = clampi(x0 - 1 + i, 0, W - 1);", "L->x[i] = clampi(x0 + i, 0, W - 1);"),
 'bh_stf16_sign': ("double sgn = ((L->wx[i] < 0.0f) != (L->wy[j] < 0.0f)) ? -1.0 : 1.0;", "double sgn = 1.0;"),
}
sel = sys.argv[1:] or list(MUTS)
for name in sel:
    old, new = MUTS[name]
    d = f'/tmp/mut2/{name}'
    shutil.rmtree(d, ignore_errors=True); os.makedirs(d)
    for sub in ('oracle','synthetic','tests'): shutil.copytree(f'{ROOT}/{sub}', f'{d}/{sub}')
    for f in os.listdir(f'{d}/oracle'):
        if f.endswith('.so'): os.remove(f'{d}/oracle/{f}')
    p = f'{d}/oracle/ctf_oracle.c'; s = open(p).read()
    if old not in s: print(name, 'PATTERN MISSING'); continue
    open(p,'w').write(s.replace(old, new, 1))
    r = subprocess.run(['python','-m','pytest','tests/test_oracle_pins.py','tests/test_oracle_bicubic.py','-q','-p','no:cacheprovider','-m','not gpu','-x'], cwd=d, capture_output=True, text=True, timeout=900)
    last = [l for l in r.stdout.splitlines() if 'passed' in l or 'failed' in l or 'error' in l.lower()]
    print(f'{name:28s}', 'KILLED' if r.returncode else 'SURVIVED', last[-1] if last else r.stdout[-300:])
