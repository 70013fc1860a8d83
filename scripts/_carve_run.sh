for c in -1 50 75 88; do SWMD_CTA_CARVE=$c bash scripts/_zz_run.sh carve$c:paper_2107_06433_b200/libswmd.so:; done
