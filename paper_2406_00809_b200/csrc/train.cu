// Batched GNP training (placeholder until the training kernels land).
#include "capi_common.hpp"

extern "C" {
#define GNPC_TRAIN_STUB(sig)                                        \
  int sig {                                                         \
    gnpc_impl::set_error("training path not built in this revision"); \
    return GNPC_EUNSUPPORTED;                                       \
  }
GNPC_TRAIN_STUB(gnpc_trainer_create(gnpc_model, int64_t, double, gnpc_trainer*))
GNPC_TRAIN_STUB(gnpc_trainer_destroy(gnpc_trainer))
GNPC_TRAIN_STUB(gnpc_forward_backward(gnpc_trainer, const double*, const double*, double*, double*, double*))
GNPC_TRAIN_STUB(gnpc_train_step(gnpc_trainer, const double*, const double*, double*))
GNPC_TRAIN_STUB(gnpc_train_step_synthetic(gnpc_trainer, uint64_t, double*))
GNPC_TRAIN_STUB(gnpc_monitor_loss(gnpc_trainer, const double*, const double*, int64_t, double*))
GNPC_TRAIN_STUB(gnpc_trainer_grad_buffer(gnpc_trainer, float**, int64_t*))
GNPC_TRAIN_STUB(gnpc_train_backward_only(gnpc_trainer, const double*, const double*, double*))
GNPC_TRAIN_STUB(gnpc_train_apply_grads(gnpc_trainer))
GNPC_TRAIN_STUB(gnpc_trainer_adam_state(gnpc_trainer, double*, double*, int64_t*))
GNPC_TRAIN_STUB(gnpc_train_preconditioner(gnpc_csr, const gnpc_train_config*, double*, double*, double*))
}
