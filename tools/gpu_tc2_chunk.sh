for c in ${CS:-4 6 8 12 16 24}; do echo "chunk $c"; WS_CONV_TC2_CHUNK=$c bash tools/gpu_c3_ab.sh base | grep -o "k_conv_tc2<0, 0>.: [0-9.]*"; done
