# ncu_digest.sh REP OUTPREFIX: turn an .ncu-rep into small text digests (details, raw, sass source gz) and delete it
rep=$1; out=$2
ncu -i $rep --page details --csv > $out.details.csv 2>/dev/null
ncu -i $rep --page raw --csv > $out.raw.csv 2>/dev/null
ncu -i $rep --page source --csv --print-source sass 2>/dev/null | gzip > $out.sass.csv.gz
rm -f $rep
