// BSP model of the parallel Suitor (scripts/micro): rounds = the critical
// path of dislodgement chains; input from scripts/micro/dump_graph.py.
// BSP simulation of the parallel Suitor: every active thread does one
// proposal per round; dislodged vertices are carried on by the dislodger.
// Reports rounds (critical path) and total proposals.
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
typedef struct { int v; double w; } C;
static int beats(double c1, int u1, double c2, int u2) { return c1 > c2 || (c1 == c2 && u1 < u2); }
int main(int argc, char** argv) {
    FILE* f = fopen(argv[1], "rb");
    long n, m; fread(&n, 8, 1, f); fread(&m, 8, 1, f);
    long* xadj = malloc(8 * (n + 1)); int* adj = malloc(4 * m); double* w = malloc(8 * m);
    fread(xadj, 8, n + 1, f); fread(adj, 4, m, f); fread(w, 8, m, f); fclose(f);
    // candidate lists sorted by the proposal order (weight desc, then smaller target via edge order)
    C* cand = malloc(sizeof(C) * m);
    for (long u = 0; u < n; ++u) {
        long lo = xadj[u], hi = xadj[u + 1];
        for (long k = lo; k < hi; ++k) { cand[k].v = adj[k]; cand[k].w = w[k]; }
        // insertion sort: best first. edge_beats(v1,c1,v2,c2,u): c1>c2 or minmax(v1,u)<minmax(v2,u)
        for (long a = lo + 1; a < hi; ++a) {
            C x = cand[a]; long b = a - 1;
            while (b >= lo) {
                C y = cand[b];
                int better;
                if (x.w != y.w) better = x.w > y.w;
                else { long a1 = x.v < u ? x.v : u, a2 = x.v < u ? u : x.v, b1 = y.v < u ? y.v : u, b2 = y.v < u ? u : y.v;
                       better = a1 < b1 || (a1 == b1 && a2 < b2); }
                if (!better) break;
                cand[b + 1] = y; --b;
            }
            cand[b + 1] = x;
        }
    }
    int* S = malloc(4 * n); double* SW = malloc(8 * n);
    for (long v = 0; v < n; ++v) S[v] = -1;
    int* cur = malloc(4 * n); long* pos = malloc(8 * n);  // per thread: carried vertex, position
    int* active = malloc(4 * n); long na = n;
    for (long t = 0; t < n; ++t) { active[t] = t; cur[t] = t; pos[t] = xadj[t]; }
    long rounds = 0, props = 0;
    // per round: each active thread tries its next candidate; conflicts at a target
    // resolved by processing in thread order (any order is a valid schedule)
    while (na > 0) {
        long nn = 0;
        for (long a = 0; a < na; ++a) {
            int t = active[a]; int u = cur[t];
            if (pos[t] >= xadj[u + 1]) continue;  // exhausted: done
            C e = cand[pos[t]]; props++;
            if (S[e.v] == -1 || beats(e.w, u, SW[e.v], S[e.v])) {
                int old = S[e.v]; S[e.v] = u; SW[e.v] = e.w;
                if (old == -1) continue; // placed, thread done
                // carry the dislodged vertex: resume after its slot of e.v
                cur[t] = old; long k = xadj[old]; while (cand[k].v != e.v) ++k; pos[t] = k + 1;
                active[nn++] = t;
            } else { pos[t]++; active[nn++] = t; }
        }
        na = nn; rounds++;
    }
    printf("n=%ld rounds=%ld proposals=%ld (%.2f per vertex)\n", n, rounds, props, (double)props / n);
    return 0;
}
