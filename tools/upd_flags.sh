for f in 7 3 2 1 0; do HELM_GB_DCGS_MASK=4 HELM_GB_UPD_FLAGS=$f python tools/dcgs_split.py 4 | sed "s/^/flags=$f /"; done
