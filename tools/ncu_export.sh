set -e
R=gpurun_out/mx_k500_full.ncu-rep
ncu -i $R --page details --csv > gpurun_out/mx_details.csv 2>/dev/null || true
ncu -i $R --page raw --csv > gpurun_out/mx_raw.csv 2>/dev/null || true
ncu -i $R --page source --csv --print-source=sass > gpurun_out/mx_source.csv 2>/dev/null || true
rm -f $R
