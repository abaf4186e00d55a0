"""Mutation check of the CPU oracle's pins (test infrastructure; not run by pytest).

Each entry is a plausible mistake in `oracle/ctf_oracle.c` (a dropped term, a wrong sign,
index or comparison, a transposed operand).  For each, the script copies oracle/, synthetic/
and tests/ to /tmp, applies the mutation, rebuilds the oracle and runs the CPU pins
(tests/test_oracle_pins.py, tests/test_oracle_pins2.py, tests/test_oracle_bicubic.py).  KILLED = some pin fails.
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
 # second batch (round 2, CPU session): lane order, coverage test, BC1 decode, RNG use,
 # Eq. 1 / C+ details, AABB / Box / Mask decisions, footprint rounding, record fields
 'ca_lane_colmajor': ("px[lane] = wx * 8 + (lane & 7);\n        py[lane] = wy * 4 + (lane >> 3);", "px[lane] = wx * 8 + (lane >> 2);\n        py[lane] = wy * 4 + (lane & 3);"),
 'cb_nan_test_on_v': ("if (isnan(uvp[0])) continue;                                   /* uncovered */", "if (isnan(uvp[1])) continue;"),
 'cc_bc1_g_replication': ("e0[1] = (g0 << 2) | (g0 >> 4);", "e0[1] = (g0 << 2) | (g0 >> 3);"),
 'cd_bc1_palette_swap': ("(code == 2) ? (2 * e0[c] + e1[c]) / 3 : (e0[c] + 2 * e1[c]) / 3;", "(code == 2) ? (e0[c] + 2 * e1[c]) / 3 : (2 * e0[c] + e1[c]) / 3;"),
 'ce_bc1_index_transposed': ("uint32_t code = (idx >> (2 * (4 * (y & 3) + (x & 3)))) & 3u;", "uint32_t code = (idx >> (2 * (4 * (x & 3) + (y & 3)))) & 3u;"),
 'cf_bc1_half_round_up': ("else out[c] = (code == 2) ? (e0[c] + e1[c]) / 2 : 0;", "else out[c] = (code == 2) ? (e0[c] + e1[c] + 1) / 2 : 0;"),
 'cg_unit24_shift9': ("return (double)(r >> 8) * (1.0 / 16777216.0);", "return (double)(r >> 9) * (1.0 / 16777216.0);"),
 'ch_stf_corner_order': ("return dx + 2 * dy;", "return 2 * dx + dy;"),
 'ci_cplus_candidates_keep_planned': ("if (in_list(P, np, cid[q])) continue;", ""),
 'cj_cplus_candidates_keep_zero_w': ("if (cw[q] == 0.0f) continue;", ""),
 'ck_eq1_Sp_weighted': ("Sp[ch] += p[ch]; plast[ch] = p[ch]; }", "Sp[ch] += dw[j] * p[ch]; plast[ch] = p[ch]; }"),
 'cl_eq1_sign': ("else c[ch] = Swp[ch] + (1.0 - Sw) * Sp[ch] / N;", "else c[ch] = Swp[ch] + (Sw - 1.0) * Sp[ch] / N;"),
 'cm_fallback_no_merge': ("dw[j] += L->w[k];\n    }\n    int all_known", "dw[j] = L->w[k];\n    }\n    int all_known"),
 'cn_partial_bit_a31': ("((uint32_t)(a < 32) << 26)", "((uint32_t)(a < 31) << 26)"),
 'co_aabb_from_id1': ("int xb = (int)(L[lane].id[3] % (uint32_t)tex->W), yb = (int)(L[lane].id[3] / (uint32_t)tex->W);", "int xb = (int)(L[lane].id[3] % (uint32_t)tex->W), yb = (int)(L[lane].id[1] / (uint32_t)tex->W);"),
 'cp_box_vs_32': ("if (F->mode == M_BOX) ok = bw * bh <= a;", "if (F->mode == M_BOX) ok = bw * bh <= 32;"),
 'cq_mask11_12': ("ok = bw <= 11 && bh <= 11 && n <= a;", "ok = bw <= 12 && bh <= 12 && n <= a;"),
 'cr_footprint_two_roundings': ("float fx = fmaf(uc, (float)W, -0.5f), fy = fmaf(vc, (float)H, -0.5f);\n    float flx = floorf(fx), fly = floorf(fy);\n    int x0 = (int)flx, y0 = (int)fly;\n    st[0]", "volatile float pxw = uc * (float)W, pyh = vc * (float)H;\n    float fx = pxw - 0.5f, fy = pyh - 0.5f;\n    float flx = floorf(fx), fly = floorf(fy);\n    int x0 = (int)flx, y0 = (int)fly;\n    st[0]"),
 'cs_uv_unclamped_low': ("float uc = fminf(fmaxf(u, 0.0f), 1.0f);\n    float vc = fminf(fmaxf(v, 0.0f), 1.0f);\n    float fx = fmaf", "float uc = fminf(u, 1.0f);\n    float vc = fminf(v, 1.0f);\n    float fx = fmaf"),
 'ct_mag_sum': ("float r2 = rx > ry ? rx : ry;\n        L->magnified", "float r2 = rx + ry;\n        L->magnified"),
 'cu_eq2_den': ("long den = 2L * (a - 1 - n);", "long den = 2L * (a - n);"),
 'cv_stf_evals_32': ("        evals = a;\n    } else if (run_fallback == FB_WC", "        evals = 32;\n    } else if (run_fallback == FB_WC"),
 'cw_unique_descending': ("return x < y ? -1 : (x > y);", "return x > y ? -1 : (x < y);"),
 'cx_4tap_evals_32': ("evals = 4 * a;", "evals = 4 * 32;"),
 'cy_cplus_target_u0': ("volatile float target = (float)u[c][2] * wsum;", "volatile float target = (float)u[c][0] * wsum;"),
 'cz_philox_ctr_frame_slot': ("uint32_t ctr[4] = { (uint32_t)px, (uint32_t)py, frame, 0u };", "uint32_t ctr[4] = { (uint32_t)px, (uint32_t)py, 0u, frame };"),
 # third batch: the latent-MLP decode (R-10), texel addressing on non-square textures,
 # the C+ plan / spare-lane loop, Mask's n <= a test, WC vs Eq. 1 dispatch
 'da_mlp_no_relu1': ("h1[j] = acc > 0 ? acc : 0;", "h1[j] = acc;"),
 'db_mlp_latent_offset': ("double gx = (x - 1.5) / 4.0, gy = (y - 1.5) / 4.0;", "double gx = (x - 2.0) / 4.0, gy = (y - 2.0) / 4.0;"),
 'dc_mlp_pos_swap': ("in[8] = ((x & 3) - 1.5) / 2.0;", "in[8] = ((y & 3) - 1.5) / 2.0;"),
 'dd_mlp_W2_transposed': ("acc += (double)W2[j * 32 + k] * h1[k];", "acc += (double)W2[k * 32 + j] * h1[k];"),
 'de_produce_row_by_H': ("int x = (int)(id % (uint32_t)t->W), y = (int)(id / (uint32_t)t->W);", "int x = (int)(id % (uint32_t)t->H), y = (int)(id / (uint32_t)t->H);"),
 'df_footprint_pitch_H': ("id[0] = (uint32_t)ya * (uint32_t)W + (uint32_t)xa;", "id[0] = (uint32_t)ya * (uint32_t)H + (uint32_t)xa;"),
 'dg_cplus_plan_unsorted': ("np = sort_unique(P, np);", ""),
 'dh_eq2_rank_not_lane': ("int l = act[oracle_eq2(j, np, a)];", "int l = oracle_eq2(j, np, a);"),
 'di_cplus_first_spare_skipped': ("for (int j = np; j < a; ++j) {", "for (int j = np + 1; j < a; ++j) {"),
 'dj_mask16_no_n_test': ("ok = bw <= 16 && bh <= 16 && n <= a;", "ok = bw <= 16 && bh <= 16;"),
 'ea_bspline_w0_scale': ("w[0] = r3 / 6.0f;", "w[0] = r3 / 3.0f;"),
 'eb_cr_w2_sign': ("w[2] = ((4.0f * s2 - 3.0f * s3) + s) * 0.5f;", "w[2] = ((4.0f * s2 - 3.0f * s3) - s) * 0.5f;"),
 'ec_bicubic_clamp_no_merge': ("L->mx[L->x[i] - L->xa] = L->mx[L->x[i] - L->xa] + L->wx[i];", "L->mx[L->x[i] - L->xa] = L->wx[i];"),
 'ed_cubic_pick_cum_signed': ("cum = cum + fabsf(w[i]);\n        if (cum > target) return i;", "cum = cum + w[i];\n        if (cum > target) return i;"),
 'ee_stf16_no_scale': ("for (int ch = 0; ch < 4; ++ch) c[ch] = sgn * (double)Sx * (double)Sy * p[ch];", "for (int ch = 0; ch < 4; ++ch) c[ch] = sgn * p[ch];"),
 'ef_positivized_same_uniform': ("volatile float target = (float)u[lobe] * Wl;", "volatile float target = (float)u[0] * Wl;"),
 'eg_fallback16_weight_transposed': ("float mw = L->mx[q] * L->my[r];", "float mw = L->mx[r] * L->my[q];"),
 'eh_blend16_transposed': ("double w = (double)L->wx[i] * (double)L->wy[j];", "double w = (double)L->wx[j] * (double)L->wy[i];"),
 'ei_tap_rows_offset': ("L->y[i] = clampi(y0 - 1 + i, 0, H - 1);", "L->y[i] = clampi(y0 + i, 0, H - 1);"),
 # bicubic C+ / records (R-26 .. R-28)
 'fa_bic_cplus_signed_weights': ("fid[nf] = id; fw[nf] = fabsf(mw); ++nf;", "fid[nf] = id; fw[nf] = mw; ++nf;"),
 'fb_bic_cplus_keep_planned': ("if (mw == 0.0f || in_list(P, np, id)) continue;", "if (mw == 0.0f) continue;"),
 'fc_bic_cplus_serves_itself': ("const int sl = act[oracle_eq2(j, np, a)];", "const int sl = cl;"),
 'fd_bic_cplus_target_u0': ("volatile float target = (float)u[cl][2] * wsum;", "volatile float target = (float)u[cl][0] * wsum;"),
 'fe_bic_rec_evals_high_bits': ("((uint32_t)((evals >> 8) & 7) << 27);", "0u;"),
 'ff_bic_n_unsaturated': ("n = nu < cap + 1 ? nu : cap + 1;", "n = nu;"),
 'fg_bic_box_cap_a': ("if (F->mode == M_BOX) ok = bw * bh <= cap;", "if (F->mode == M_BOX) ok = bw * bh <= a;"),
 'dk_wc_as_eq1': ("if (L[lane].active) blend_fallback(tex, &L[lane], plist, np, run_fallback == FB_WC, col[lane]);", "if (L[lane].active) blend_fallback(tex, &L[lane], plist, np, 0, col[lane]);"),
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
    r = subprocess.run(['python','-m','pytest','tests/test_oracle_pins.py','tests/test_oracle_pins2.py','tests/test_oracle_bicubic.py','-q','-p','no:cacheprovider','-m','not gpu','-x'], cwd=d, capture_output=True, text=True, timeout=900)
    last = [l for l in r.stdout.splitlines() if 'passed' in l or 'failed' in l or 'error' in l.lower()]
    print(f'{name:28s}', 'KILLED' if r.returncode else 'SURVIVED', last[-1] if last else r.stdout[-300:])
