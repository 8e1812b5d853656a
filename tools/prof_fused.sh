bash tools/prof_one.sh fz k_modup_cols k_ntt_rows_ip k_ntt_rows_final k_moddown_bconv
