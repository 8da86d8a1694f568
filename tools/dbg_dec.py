import sys, numpy as np
sys.path.insert(0, '.')
import paper_2105_12912_b200 as lzb
rng = np.random.default_rng(2026)
books = []
g = np.array([int(1e6 * 0.55 ** abs(i - 512)) + 1 for i in range(1024)], np.int64)
books.append(g)
books.append(rng.integers(50, 200, 300).astype(np.int64))
books.append(np.array([2 ** (20 - i // 3) for i in range(60)], np.int64))
books.append(np.array([1000, 1], np.int64))
for bi, counts in enumerate(books):
    p = counts / counts.sum()
    for n in (1, 2, 63, 64, 65, 2047, 2048, 2049, 4095, 4096, 4097, 40000, 250_000):
        stream = rng.choice(len(counts), size=n, p=p).astype(np.uint32)
        bk = lzb.Codebook.from_counts(np.bincount(stream, minlength=len(counts)))
        bs = lzb.encode(stream, bk)
        try:
            d = lzb.decode(bs, bk)
            ok = np.array_equal(d, stream)
            msg = "ok" if ok else "MISMATCH first=%d" % int(np.argmax(d != stream))
        except Exception as ex:
            msg = "EXC " + str(ex)
        print(bi, n, bs.bit_len, int(bk.lengths.max()), msg, flush=True)
