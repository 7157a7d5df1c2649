#!/bin/bash
# quorum sweep of the exact walk on the steady-state C3 event (WS_FLUCT_QUORUM)
for q in ${QS:-5 6 7 8 9 10}; do echo "quorum $q"; WS_FLUCT_QUORUM=$q bash tools/gpu_c3_ab.sh base | grep -o "k_fluct_walk.: [0-9.]*"; done
