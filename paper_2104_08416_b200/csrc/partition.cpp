// partition.cpp -- multi-GPU partition of the Hilbert-ordered mesh (product path,
// SURVEY.md §8e).  Every rank holds the full reordered connectivity (each rank
// runs the same deterministic sem_mesh_reorder), so no setup collective is
// needed beyond the NCCL unique id.
//
// Rank r owns elements [floor(rE/G), floor((r+1)E/G)) of the global order.
// Because the order follows a Hilbert curve, a rank's elements form a compact
// region and only nodes on the region's border are touched by other ranks.
#include <algorithm>
#include <cstring>

#include "sem_internal.h"

namespace sem {

bool build_partition(const int32_t *mu, int64_t E, int Np, int64_t N, int rank, int world,
                     Partition &P, std::string &err) {
    if (world < 1 || world > 32 || rank < 0 || rank >= world) {
        err = "build_partition: world size must be in [1, 32]";
        return false;
    }
    P = Partition();
    P.rank = rank;
    P.world = world;
    P.e0 = (int64_t)((__int128)rank * E / world);
    P.e1 = (int64_t)((__int128)(rank + 1) * E / world);
    if (P.e1 <= P.e0) {
        err = "build_partition: rank " + std::to_string(rank) + " has no elements";
        return false;
    }
    if (world == 1) {  // one rank: everything is local, nothing is exchanged
        P.loc2glob.resize(N);
        for (int64_t g = 0; g < N; g++) P.loc2glob[g] = (int32_t)g;
        P.mu_local.assign(mu, mu + E * Np);
        P.remote.assign(N, 0);
        P.owned.assign(N, 1);
        P.nbr_off.assign(1, 0);
        P.sum_start.assign(1, 0);
        return true;
    }
    // Which ranks touch each node (bit mask; world <= 32).
    std::vector<uint32_t> mask(N, 0u);
    for (int q = 0; q < world; q++) {
        const int64_t a = (int64_t)((__int128)q * E / world), b = (int64_t)((__int128)(q + 1) * E / world);
        const uint32_t bit = 1u << q;
        for (int64_t i = a * Np; i < b * Np; i++) mask[mu[i]] |= bit;
    }
    const uint32_t me = 1u << rank;
    // Local nodes in ascending global id.
    std::vector<int32_t> g2l(N, -1);
    for (int64_t g = 0; g < N; g++)
        if (mask[g] & me) {
            g2l[g] = (int32_t)P.loc2glob.size();
            P.loc2glob.push_back((int32_t)g);
        }
    const int64_t NL = (int64_t)P.loc2glob.size();
    P.remote.assign(NL, 0);
    P.owned.assign(NL, 0);
    for (int64_t l = 0; l < NL; l++) {
        const uint32_t m = mask[P.loc2glob[l]];
        P.remote[l] = (m & ~me) != 0;
        P.owned[l] = (m & (me - 1)) == 0;  // no lower rank touches it
        if (P.remote[l]) P.if_local.push_back((int32_t)l);
    }
    P.mu_local.resize((size_t)(P.e1 - P.e0) * Np);
    for (int64_t i = P.e0 * Np, k = 0; i < P.e1 * Np; i++, k++) P.mu_local[k] = g2l[mu[i]];
    // Neighbours and per-neighbour lists (ascending global id == ascending interface index).
    const int64_t nif = (int64_t)P.if_local.size();
    uint32_t nbr_mask = 0;
    for (int64_t i = 0; i < nif; i++) nbr_mask |= mask[P.loc2glob[P.if_local[i]]];
    nbr_mask &= ~me;
    for (int q = 0; q < world; q++)
        if (nbr_mask & (1u << q)) P.nbr.push_back(q);
    const int nn = (int)P.nbr.size();
    P.nbr_off.assign(nn + 1, 0);
    std::vector<std::vector<int32_t>> pos_in(nn, std::vector<int32_t>(nif, -1));
    for (int k = 0; k < nn; k++) {
        const uint32_t bit = 1u << P.nbr[k];
        int32_t cnt = 0;
        for (int64_t i = 0; i < nif; i++)
            if (mask[P.loc2glob[P.if_local[i]]] & bit) {
                pos_in[k][i] = P.nbr_off[k] + cnt;
                P.send_if.push_back((int32_t)i);
                cnt++;
            }
        P.nbr_off[k + 1] = P.nbr_off[k] + cnt;
    }
    // Summation order per interface node: all touching ranks, ascending.
    P.sum_start.assign(nif + 1, 0);
    for (int64_t i = 0; i < nif; i++) {
        const uint32_t m = mask[P.loc2glob[P.if_local[i]]];
        for (int q = 0; q < world; q++) {
            if (!(m & (1u << q))) continue;
            if (q == rank) {
                P.sum_src.push_back((int32_t)i);
            } else {
                const int k = (int)(std::lower_bound(P.nbr.begin(), P.nbr.end(), q) - P.nbr.begin());
                P.sum_src.push_back((int32_t)(nif + pos_in[k][i]));
            }
        }
        P.sum_start[i + 1] = (int32_t)P.sum_src.size();
    }
    return true;
}

}  // namespace sem
