#include <stdio.h>
#include "vqhull_b200.h"
int main(void) {
    double xs[] = {0, 4, 4, 0, 2, 0}, ys[] = {0, 0, 4, 4, 2, 0};
    size_t idx[6], cnt = 0;
    fprintf(stderr, "calling\n");
    int rc = vqhull_compute(xs, ys, 6, 1, idx, &cnt);
    fprintf(stderr, "rc=%d cnt=%zu first=%zu\n", rc, cnt, idx[0]);
    double x1[] = {0}, y1[] = {0};
    rc = vqhull_compute(x1, y1, 1, 1, idx, &cnt);
    fprintf(stderr, "single rc=%d cnt=%zu\n", rc, cnt);
    return 0;
}
