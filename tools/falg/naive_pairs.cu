// naive per-pair bodies (libdevice exp), one loop iteration = one pair
struct C { double kx, kt, ks, om, lb, ls, ab, bs; };
// ordered pair, rate pass (both terms, self gated by time order)
extern "C" __global__ void ord_rate(const double2* x, const double* t, int N, C c, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= N) return;
  double2 xi = x[i]; double ti = t[i], M = 0, X = 0;
  for (int j = 0; j < N; ++j) {
    double dx = x[j].x - xi.x, dy = x[j].y - xi.y, r2 = dx*dx + dy*dy, dt = ti - t[j];
    if (dt != 0.0) M += exp(c.lb + c.kx * r2 + c.kt * dt * dt);
    if (dt > 0.0) X += exp(c.ls + c.ks * r2 - c.om * dt);
  }
  out[2*i] = M; out[2*i+1] = X;
}
// unordered pair, rate pass: each pair once, mu to both rows, xi to the later one
extern "C" __global__ void uno_rate(const double2* x, const double* t, int N, C c, double* acc_i, double* acc_j) {
  int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= N) return;
  double2 xi = x[i]; double ti = t[i], Mi = 0, Xi = 0;
  for (int j = i + 1; j < N; ++j) {
    double dx = x[j].x - xi.x, dy = x[j].y - xi.y, r2 = dx*dx + dy*dy, dt = ti - t[j];
    double m = dt != 0.0 ? exp(c.lb + c.kx * r2 + c.kt * dt * dt) : 0.0;
    double s = dt != 0.0 ? exp(c.ls + c.ks * r2 - c.om * fabs(dt)) : 0.0;
    Mi += m; acc_j[2*j] += m;
    if (dt > 0.0) Xi += s; else acc_j[2*j+1] += s;
  }
  acc_i[2*i] = Mi; acc_i[2*i+1] = Xi;
}
// unordered pair, gradient pass: c = ab e_b (rho_i + rho_j) + bs e_s rho_later; g_i += c dx, g_j -= c dx
extern "C" __global__ void uno_grad(const double2* x, const double* t, const double* rho, int N, C c, double2* gj) {
  int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= N) return;
  double2 xi = x[i]; double ti = t[i], ri = rho[i], gx = 0, gy = 0;
  for (int j = i + 1; j < N; ++j) {
    double dx = x[j].x - xi.x, dy = x[j].y - xi.y, r2 = dx*dx + dy*dy, dt = ti - t[j];
    double cc = 0.0;
    if (dt != 0.0) {
      double eb = exp(c.lb + c.kx * r2 + c.kt * dt * dt);
      double es = exp(c.ls + c.ks * r2 - c.om * fabs(dt));
      cc = c.ab * eb * (ri + rho[j]) + c.bs * es * (dt > 0.0 ? ri : rho[j]);
    }
    gx += cc * dx; gy += cc * dy; gj[j].x -= cc * dx; gj[j].y -= cc * dy;
  }
  gj[i].x += gx; gj[i].y += gy;
}
// ordered pair, gradient pass (as SURVEY: both terms per ordered pair)
extern "C" __global__ void ord_grad(const double2* x, const double* t, const double* rho, int N, C c, double2* g) {
  int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= N) return;
  double2 xi = x[i]; double ti = t[i], ri = rho[i], gx = 0, gy = 0;
  for (int j = 0; j < N; ++j) {
    double dx = x[j].x - xi.x, dy = x[j].y - xi.y, r2 = dx*dx + dy*dy, dt = ti - t[j];
    if (dt != 0.0) {
      double eb = exp(c.lb + c.kx * r2 + c.kt * dt * dt);
      double es = exp(c.ls + c.ks * r2 - c.om * fabs(dt));
      double cc = c.ab * eb * (ri + rho[j]) + c.bs * es * (dt > 0.0 ? ri : rho[j]);
      gx += cc * dx; gy += cc * dy;
    }
  }
  g[i].x = gx; g[i].y = gy;
}
