source <(head -14 scripts/ab_c4.sh)
run def
run lcu16 PLSS_LIB=paper_2207_07615_b200/libplss_lcu16.so
run lcu12 PLSS_LIB=paper_2207_07615_b200/libplss_lcu12.so
run def2
BARGS="--workload C4alt"
run alt_def
run alt_lcu16 PLSS_LIB=paper_2207_07615_b200/libplss_lcu16.so
run alt_lcu12 PLSS_LIB=paper_2207_07615_b200/libplss_lcu12.so
