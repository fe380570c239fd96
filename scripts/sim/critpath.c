/* Critical-path model of the exact wavefront sweep (analysis tool, not
 * product): runs the reference order (oracle/liboracle.so's best_candidate,
 * host fields from a .bin dump) with the 8-neighbour dirty rule, and for each
 * pass computes the earliest finish time of every node when
 *   time(n) = cost(n) + max(time of its new neighbours in this pass,
 *                          time of its 3x3 neighbourhood in the previous pass)
 * plus the iteration-decision barrier (passes 1..3 of iteration it+1 wait for
 * all of iteration it).  cost = td for a dirty node, tc for a clean one.
 * Prints the modelled solve time for several (td, tc).
 *   cc -O2 critpath.c -L../../oracle -loracle -lm -o critpath
 *   ./critpath fields.bin N */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include "../../oracle/oracle.h"

static int R, C;
static void lw(int dir, int L, int W, int* r, int* c) {
    switch (dir) {
        case 0: *r = W; *c = L; break;
        case 1: *r = L; *c = C - 1 - W; break;
        case 2: *r = R - 1 - W; *c = C - 1 - L; break;
        default: *r = R - 1 - L; *c = W; break;
    }
}
#define NC 5
int main(int argc, char** argv) {
    int N = atoi(argv[2]);
    R = C = N;
    size_t n = (size_t)N * N;
    double* F = malloc(5 * n * sizeof(double));
    FILE* f = fopen(argv[1], "rb");
    if (fread(F, sizeof(double), 5 * n, f) != 5 * n) return 1;
    fclose(f);
    double h = 1.0 / N;
    double *g11 = F, *g12 = F + n, *g22 = F + 2 * n, *b1 = F + 3 * n, *b2 = F + 4 * n;
    double* T = malloc(n * sizeof(double));
    uint8_t* st = malloc(n);
    for (size_t i = 0; i < n; ++i) { T[i] = 1e10; st[i] = 254; }
    size_t s0 = (size_t)(N / 2) * N + N / 2;
    T[s0] = 0.0; st[s0] = 255;
    /* k = 0..2: cost by dirtiness (td / tc); k = 3: cost 1 only for nodes that change (optimistic) */
    /* k = 4: depth-2 speculation: a node whose critical predecessors (same
       line W-1, previous line W+1) did not change costs 0.45, otherwise 1.1;
       clean nodes 0.25 (validation + barrier) */
    double td[NC] = {1, 1, 1, 1, 1}, tc[NC] = {1, 0.5, 0.0, 0.0, 0.25};
    uint8_t* chg = calloc(n, 1);
    double* tp[NC]; double* tq[NC]; double itmax[NC], gate[NC], fin[NC];
    for (int k = 0; k < NC; ++k) {
        tp[k] = calloc(n, sizeof(double)); tq[k] = calloc(n, sizeof(double));
        itmax[k] = 0; gate[k] = 0; fin[k] = 0;
    }
    double* prev = malloc(n * sizeof(double));
    long long dirty_tot = 0, nodes_tot = 0;
    for (int it = 0; it < 50; ++it) {
        memcpy(prev, T, n * sizeof(double));
        double pass_start_gate[NC];
        for (int q = 0; q < 4; ++q) {
            int dir = q;
            unsigned S = (unsigned)(it * 4 + q) & 0xff, Sp = (S - 1) & 0xff;
            int NL = (dir & 1) ? R : C, NW = (dir & 1) ? C : R;
            /* passes q>0 of iteration it>0 wait for iteration it-1's decision */
            for (int k = 0; k < NC; ++k) pass_start_gate[k] = (q > 0 && it > 0) ? gate[k] : 0.0;
            long long dirty = 0;
            for (int L = 0; L < NL; ++L) {
                for (int W = 0; W < NW; ++W) {
                    int r, c;
                    lw(dir, L, W, &r, &c);
                    size_t i = (size_t)r * C + c;
                    int d = 0;
                    for (int dr = -1; dr <= 1; ++dr)
                        for (int dc = -1; dc <= 1; ++dc) {
                            if (!dr && !dc) continue;
                            int rr = r + dr, cc = c + dc;
                            if (rr < 0 || rr >= R || cc < 0 || cc >= C) continue;
                            uint8_t s = st[(size_t)rr * C + cc];
                            if (s == S || s == Sp) d = 1;
                        }
                    if (i == s0) d = 0;
                    chg[i] = 0;
                    int changed = 0;
                    /* critical predecessors changed in this pass? */
                    int crit = 0;
                    {
                        int LL[2] = {L, L - 1}, WW[2] = {W - 1, W + 1};
                        for (int e = 0; e < 2; ++e) {
                            if (LL[e] < 0 || WW[e] < 0 || WW[e] >= NW) continue;
                            int r2, c2; lw(dir, LL[e], WW[e], &r2, &c2);
                            if (chg[(size_t)r2 * C + c2]) crit = 1;
                        }
                    }
                    if (d) {
                        ++dirty;
                        orc_candidate cand = orc_best_candidate(r, c, R, C, h, T, g11, g12, g22, b1, b2);
                        if (cand.found && cand.t0 < T[i]) { T[i] = cand.t0; st[i] = (uint8_t)S; changed = 1; }
                        chg[i] = (uint8_t)changed;
                    }
                    /* timing: new neighbours in this pass = (L-1, W-1..W+1), (L, W-1) */
                    for (int k = 0; k < NC; ++k) {
                        double m = pass_start_gate[k];
                        int LL[4] = {L - 1, L - 1, L - 1, L}, WW[4] = {W - 1, W, W + 1, W - 1};
                        for (int e = 0; e < 4; ++e) {
                            if (LL[e] < 0 || WW[e] < 0 || WW[e] >= NW) continue;
                            int r2, c2; lw(dir, LL[e], WW[e], &r2, &c2);
                            double v = tq[k][(size_t)r2 * C + c2];
                            if (v > m) m = v;
                        }
                        for (int dr = -1; dr <= 1; ++dr)
                            for (int dc = -1; dc <= 1; ++dc) {
                                int rr = r + dr, cc = c + dc;
                                if (rr < 0 || rr >= R || cc < 0 || cc >= C) continue;
                                double v = tp[k][(size_t)rr * C + cc];
                                if (v > m) m = v;
                            }
                        double cost;
                        if (k == 3) cost = changed ? 1.0 : 0.0;
                        else if (k == 4) cost = !d ? tc[4] : (crit ? 1.1 : 0.45);
                        else cost = d ? td[k] : tc[k];
                        tq[k][i] = m + cost;
                    }
                }
            }
            dirty_tot += dirty; nodes_tot += n;
            memset(chg, 0, n);
            for (int k = 0; k < NC; ++k) {
                double mx = 0;
                for (size_t i = 0; i < n; ++i) if (tq[k][i] > mx) mx = tq[k][i];
                if (q == 3) gate[k] = mx;
                fin[k] = mx > fin[k] ? mx : fin[k];
                double* t = tp[k]; tp[k] = tq[k]; tq[k] = t;
            }
            fprintf(stderr, "it %d pass %d dirty %.3f  finish(steps) tc=1:%.0f tc=.5:%.0f tc=0:%.0f changed-only:%.0f spec2:%.0f\n", it, q,
                    (double)dirty / n, fin[0], fin[1], fin[2], fin[3], fin[4]);
        }
        double md = 0;
        for (size_t i = 0; i < n; ++i) { double dd = fabs(T[i] - prev[i]); if (dd > md) md = dd; }
        if (md < 1e-6) { fprintf(stderr, "converged K=%d\n", it + 1); break; }
    }
    printf("N=%d dirty fraction %.3f; critical path in node-steps: tc=1 %.0f, tc=0.5 %.0f, tc=0 %.0f, changed-only %.0f, spec2 %.0f\n", N,
           (double)dirty_tot / nodes_tot, fin[0], fin[1], fin[2], fin[3], fin[4]);
    return 0;
}
