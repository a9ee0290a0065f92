import sys; sys.path.insert(0, '.')
import paper_2508_18556_b200 as mig
n = int(sys.argv[1])
masks = sorted({((1 << L) - 1) << s for L, step in [(1, 1), (2, 2), (4, 4), (6, 6), (12, 12), (24, 24)]
                for s in range(0, n - L + 1, step)} | {0b111 << s for s in range(0, n - 2, 4)})
fcr, fl, info = mig.mig_reachability(n, masks)
print(n, info)
