for d in 0 1 2 3 4; do
  echo "dbg=$d"; CARVE_DP_DBG=$d timeout 60 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, paper_2410_21207_b200 as cv
e=(np.arange(14,dtype=np.float64).reshape(2,7)*7)%5
try: print(cv.dp_seam(e).seam)
except Exception as ex: print('ERR', ex)
"
done
