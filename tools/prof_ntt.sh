bash tools/prof_one.sh pipe k_ntt_rows_pipe k_ntt_cols_pipe
HY_NTT_PIPE=0 bash tools/prof_one.sh old k_ntt_rows k_ntt_cols256
